import sys; sys.path.insert(0, "/root/repo")
import bench
class A: seed = 42; iters = 20
print(bench.sum_product_f32_rate(A(), B=2048))
