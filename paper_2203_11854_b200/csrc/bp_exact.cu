// EXACT-mode flooding BP (ldpc.py:86-172) on a generic check-major CSR graph.
//
// Reproduces the reference's arithmetic bit for bit for min-sum and
// scaled-min-sum, and its precision pattern for sum-product:
//   * f32 input: posterior `total` is f32, messages c2v are f64 from the
//     first iteration on (sign_excl is float64, ldpc.py:136); iteration 1
//     computes v2c, |v2c|, phi and the check phi-sums in f32;
//   * f64 input: everything f64;
//   * numpy add.reduceat order: x0 + pairwise_sum(x1..), pairwise_sum
//     starting from -0.0 and 8-way unrolled for 8..128 terms;
//   * total = clip(cast(channel + sum), +-40);  syndrome on signbit(total)
//     after each iteration, converged rows frozen (ldpc.py:155-167).
//
// Layout: everything batch-innermost ([edge][b], [var][b]) so a warp of
// threads = 32 consecutive codewords makes every access coalesced.  Kernels
// per iteration: check update, variable update, syndrome, freeze.
#include <math.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace lsb {

// nodes up to this degree keep their edge values in registers / local
// memory; higher degrees stream over their edges twice (same results)
constexpr int kExactMaxDeg = 64;

template <typename T>
__device__ __forceinline__ T pairwise(const T *x, int n) {
  // numpy pairwise_sum for n <= 128 (degrees are capped at kExactMaxDeg)
  if (n < 8) {
    T r = (T)-0.0;
    for (int i = 0; i < n; ++i) r = r + x[i];
    return r;
  }
  T r0 = x[0], r1 = x[1], r2 = x[2], r3 = x[3], r4 = x[4], r5 = x[5], r6 = x[6], r7 = x[7];
  int i;
  for (i = 8; i < n - (n % 8); i += 8) {
    r0 = r0 + x[i]; r1 = r1 + x[i + 1]; r2 = r2 + x[i + 2]; r3 = r3 + x[i + 3];
    r4 = r4 + x[i + 4]; r5 = r5 + x[i + 5]; r6 = r6 + x[i + 6]; r7 = r7 + x[i + 7];
  }
  T res = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
  for (; i < n; ++i) res = res + x[i];
  return res;
}

template <typename T>
__device__ __forceinline__ T segsum(const T *x, int n) {
  return n == 1 ? x[0] : x[0] + pairwise(x + 1, n - 1);
}

// numpy pairwise_sum of term(off..off+n-1), n <= 128, without storing the terms
template <typename T, class F>
__device__ T pairwise_block(int off, int n, const F &term) {
  if (n < 8) {
    T r = (T)-0.0;
    for (int i = 0; i < n; ++i) r = r + term(off + i);
    return r;
  }
  T r0 = term(off), r1 = term(off + 1), r2 = term(off + 2), r3 = term(off + 3), r4 = term(off + 4),
    r5 = term(off + 5), r6 = term(off + 6), r7 = term(off + 7);
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
    r0 = r0 + term(off + i); r1 = r1 + term(off + i + 1); r2 = r2 + term(off + i + 2); r3 = r3 + term(off + i + 3);
    r4 = r4 + term(off + i + 4); r5 = r5 + term(off + i + 5); r6 = r6 + term(off + i + 6); r7 = r7 + term(off + i + 7);
  }
  T res = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
  for (; i < n; ++i) res = res + term(off + i);
  return res;
}

// any n: above 128 terms numpy splits the block in two halves (n/2 rounded
// down to a multiple of 8) and recurses; the recursion is walked here with
// an explicit stack (device recursion would overflow the thread stack)
template <typename T, class F>
__device__ T pairwise_stream(int off, int n, const F &term) {
  if (n <= 128) return pairwise_block<T>(off, n, term);
  struct Frame {
    int off, n, n2, state;
    T left;
  };
  Frame st[24];  // depth log2(n / 128) + 1
  int sp = 0;
  st[0] = Frame{off, n, 0, 0, (T)0};
  T ret = (T)0;
  bool have = false;  // `ret` holds the value of the frame just finished
  while (sp >= 0) {
    Frame &f = st[sp];
    if (have) {
      if (f.state == 1) {  // left half done: evaluate the right half
        f.left = ret;
        f.state = 2;
        have = false;
        st[sp + 1] = Frame{f.off + f.n2, f.n - f.n2, 0, 0, (T)0};
        ++sp;
      } else {  // both halves done
        ret = f.left + ret;
        --sp;
      }
      continue;
    }
    if (f.n <= 128) {
      ret = pairwise_block<T>(f.off, f.n, term);
      have = true;
      --sp;
      continue;
    }
    int n2 = f.n / 2;
    n2 -= n2 % 8;
    f.n2 = n2;
    f.state = 1;
    st[sp + 1] = Frame{f.off, n2, 0, 0, (T)0};
    ++sp;
  }
  return ret;
}

// x0 + pairwise(x1..x_{n-1}) (numpy add.reduceat of one segment)
template <typename T, class F>
__device__ T segsum_stream(int n, const F &term) {
  return n == 1 ? term(0) : term(0) + pairwise_stream<T>(1, n - 1, term);
}

__device__ __forceinline__ double phi_d(double x) {
  x = fmin(fmax(x, 1e-12), 40.0);
  return -log(tanh(x / 2.0));
}
__device__ __forceinline__ float phi_f(float x) {
  x = fminf(fmaxf(x, 1e-12f), 40.0f);
  return -logf(tanhf(x / 2.0f));
}

// ---------------------------------------------------------------- init
template <typename T>
__global__ void k_ex_init(const T *__restrict__ llr, int64_t B, int64_t n, T *__restrict__ chan,
                          T *__restrict__ total) {
  // [B, n] -> [n, B] through a 32x32 smem tile
  __shared__ T tile[32][33];
  const int64_t v0 = blockIdx.x * 32, b0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    int64_t b = b0 + r, v = v0 + threadIdx.x;
    if (b < B && v < n) tile[r][threadIdx.x] = llr[b * n + v];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    int64_t v = v0 + r, b = b0 + threadIdx.x;
    if (b < B && v < n) {
      T c = -tile[threadIdx.x][r];
      chan[v * B + b] = c;
      total[v * B + b] = c;
    }
  }
}

template <typename T>
__global__ void k_ex_output(const T *__restrict__ total, int64_t B, int64_t n, T *__restrict__ out,
                            uint8_t *__restrict__ hard) {
  __shared__ T tile[32][33];
  const int64_t v0 = blockIdx.x * 32, b0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    int64_t v = v0 + r, b = b0 + threadIdx.x;
    if (b < B && v < n) tile[r][threadIdx.x] = total[v * B + b];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    int64_t b = b0 + r, v = v0 + threadIdx.x;
    if (b < B && v < n) {
      T o = -tile[threadIdx.x][r];
      if (out) out[b * n + v] = o;
      if (hard) hard[b * n + v] = o > (T)0;
    }
  }
}

// ---------------------------------------------------------------- check update
template <typename T, int VARIANT>
__global__ void k_ex_check(const int32_t *__restrict__ cptr, const int32_t *__restrict__ cvar, int64_t m,
                           int64_t B, const T *__restrict__ total, double *__restrict__ c2v,
                           const uint8_t *__restrict__ active, int first_f32, double alpha) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= B || !active[b]) return;
  double v2c[kExactMaxDeg];
  for (int64_t c = blockIdx.y; c < m; c += gridDim.y) {
    const int e0 = cptr[c], d = cptr[c + 1] - e0;
    if (d > kExactMaxDeg) {
      // high-degree check: the same arithmetic in two streaming passes over
      // the edges (each v2c recomputed from total and the not yet
      // overwritten c2v of its own edge), no per-check array
      auto v2c_at = [&](int j) -> double {
        const int64_t e = e0 + j;
        return (double)total[(int64_t)cvar[e] * B + b] - c2v[e * B + b];
      };
      int par = 0;
      for (int j = 0; j < d; ++j) par ^= signbit(v2c_at(j)) ? 1 : 0;
      if (VARIANT == LS_SUM_PRODUCT) {
        if (first_f32) {
          auto pmf = [&](int j) -> float { return phi_f(fabsf((float)v2c_at(j))); };
          const float ps = segsum_stream<float>(d, pmf);
          for (int j = 0; j < d; ++j) {
            const double x = v2c_at(j);
            float me = phi_f(fmaxf(ps - phi_f(fabsf((float)x)), 1e-12f));
            me = fminf(fmaxf(me, 0.0f), 30.0f);
            const int neg = par ^ (signbit(x) ? 1 : 0);
            c2v[(e0 + j) * B + b] = (neg ? -1.0 : 1.0) * (double)me;
          }
        } else {
          auto pmd = [&](int j) -> double { return phi_d(fabs(v2c_at(j))); };
          const double ps = segsum_stream<double>(d, pmd);
          for (int j = 0; j < d; ++j) {
            const double x = v2c_at(j);
            double me = phi_d(fmax(ps - phi_d(fabs(x)), 1e-12));
            me = fmin(fmax(me, 0.0), 30.0);
            const int neg = par ^ (signbit(x) ? 1 : 0);
            c2v[(e0 + j) * B + b] = (neg ? -1.0 : 1.0) * me;
          }
        }
      } else {
        // multiset minimum pair + first argmin == _segment_min2's rule
        // (ldpc.py:65-74): a tie makes the runner-up equal to min1
        double mn1 = INFINITY, mn2 = INFINITY;
        int arg = 0;
        for (int j = 0; j < d; ++j) {
          const double a = fabs(v2c_at(j));
          if (a < mn1) {
            mn2 = mn1;
            mn1 = a;
            arg = j;
          } else if (a < mn2) {
            mn2 = a;
          }
        }
        for (int j = 0; j < d; ++j) {
          const double x = v2c_at(j);
          const int neg = par ^ (signbit(x) ? 1 : 0);
          c2v[(e0 + j) * B + b] = __dmul_rn(neg ? -alpha : alpha, j == arg ? mn2 : mn1);
        }
      }
      continue;
    }
    int par = 0;
    for (int j = 0; j < d; ++j) {
      const int64_t e = e0 + j;
      const double t = (double)total[(int64_t)cvar[e] * B + b];
      v2c[j] = t - c2v[e * B + b];
      par ^= signbit(v2c[j]) ? 1 : 0;
    }
    if (VARIANT == LS_SUM_PRODUCT) {
      if (first_f32) {
        float pm[kExactMaxDeg];
        for (int j = 0; j < d; ++j) pm[j] = phi_f(fabsf((float)v2c[j]));
        const float ps = segsum(pm, d);
        for (int j = 0; j < d; ++j) {
          float me = phi_f(fmaxf(ps - pm[j], 1e-12f));
          me = fminf(fmaxf(me, 0.0f), 30.0f);
          const int neg = par ^ (signbit(v2c[j]) ? 1 : 0);
          c2v[(e0 + j) * B + b] = (neg ? -1.0 : 1.0) * (double)me;
        }
      } else {
        double pm[kExactMaxDeg];
        for (int j = 0; j < d; ++j) pm[j] = phi_d(fabs(v2c[j]));
        const double ps = segsum(pm, d);
        for (int j = 0; j < d; ++j) {
          double me = phi_d(fmax(ps - pm[j], 1e-12));
          me = fmin(fmax(me, 0.0), 30.0);
          const int neg = par ^ (signbit(v2c[j]) ? 1 : 0);
          c2v[(e0 + j) * B + b] = (neg ? -1.0 : 1.0) * me;
        }
      }
    } else {
      // _segment_min2 tie rule (ldpc.py:65-74): unique argmin gets min2
      double mn1 = INFINITY, mn2 = INFINITY;
      for (int j = 0; j < d; ++j) mn1 = fmin(mn1, fabs(v2c[j]));
      int cnt = 0;
      for (int j = 0; j < d; ++j) {
        const double a = fabs(v2c[j]);
        if (a == mn1) ++cnt;
        else mn2 = fmin(mn2, a);
      }
      for (int j = 0; j < d; ++j) {
        const double a = fabs(v2c[j]);
        const double ex = (a == mn1 && cnt == 1) ? mn2 : mn1;
        const int neg = par ^ (signbit(v2c[j]) ? 1 : 0);
        c2v[(e0 + j) * B + b] = __dmul_rn(neg ? -alpha : alpha, ex);
      }
    }
  }
}

// ---------------------------------------------------------------- variable update
template <typename T>
__global__ void k_ex_var(const int32_t *__restrict__ vptr, const int32_t *__restrict__ vedge, int64_t n,
                         int64_t B, const T *__restrict__ chan, T *__restrict__ total,
                         const double *__restrict__ c2v, const uint8_t *__restrict__ active) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= B || !active[b]) return;
  double x[kExactMaxDeg];
  for (int64_t v = blockIdx.y; v < n; v += gridDim.y) {
    const int p0 = vptr[v], d = vptr[v + 1] - p0;
    const int64_t o = v * B + b;
    if (d == 0) {
      total[o] = chan[o];
      continue;
    }
    double s;
    if (d > kExactMaxDeg) {
      s = segsum_stream<double>(d, [&](int j) -> double { return c2v[(int64_t)vedge[p0 + j] * B + b]; });
    } else {
      for (int j = 0; j < d; ++j) x[j] = c2v[(int64_t)vedge[p0 + j] * B + b];
      s = segsum(x, d);
    }
    T t = (T)((double)chan[o] + s);
    t = t < (T)-40.0 ? (T)-40.0 : (t > (T)40.0 ? (T)40.0 : t);
    total[o] = t;
  }
}

// ---------------------------------------------------------------- early stop
template <typename T>
__global__ void k_ex_syndrome(const int32_t *__restrict__ cptr, const int32_t *__restrict__ cvar, int64_t m,
                              int64_t B, const T *__restrict__ total, const uint8_t *__restrict__ active,
                              uint8_t *__restrict__ unsat) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= B || !active[b]) return;
  for (int64_t c = blockIdx.y; c < m; c += gridDim.y) {
    int syn = 0;
    for (int e = cptr[c]; e < cptr[c + 1]; ++e) syn ^= signbit(total[(int64_t)cvar[e] * B + b]) ? 1 : 0;
    if (syn) unsat[b] = 1;
  }
}

__global__ void k_ex_freeze(int64_t B, uint8_t *__restrict__ active, uint8_t *__restrict__ unsat,
                            int32_t *__restrict__ iters, int it) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= B) return;
  if (active[b] && !unsat[b]) {
    active[b] = 0;
    iters[b] = it + 1;
  }
  unsat[b] = 0;
}

__global__ void k_fill_u8(uint8_t *p, int64_t n, uint8_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}
__global__ void k_fill_i32(int32_t *p, int64_t n, int32_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

template <typename T>
static int run_exact(const ls_graph *g, const T *llr, int64_t B, int num_iter, int variant, double scale,
                     int early_stop, T *out, uint8_t *hard, int32_t *iters_used, cudaStream_t s) {
  const int64_t n = g->n, m = g->m, E = g->E;
  T *chan = nullptr, *total = nullptr;
  double *c2v = nullptr;
  uint8_t *flags = nullptr;
  int32_t *iters = nullptr;
  cudaError_t e;
  retain_pool_memory();  // the workspace is [E, B] f64, ~1 GB for 1024 BG1 Z=384 codewords
#define LS_TRY(x)                                \
  do {                                           \
    e = (x);                                     \
    if (e != cudaSuccess) goto fail_;            \
  } while (0)
  LS_TRY(cudaMallocAsync((void **)&chan, sizeof(T) * n * B, s));
  LS_TRY(cudaMallocAsync((void **)&total, sizeof(T) * n * B, s));
  LS_TRY(cudaMallocAsync((void **)&c2v, sizeof(double) * std::max<int64_t>(E, 1) * B, s));
  LS_TRY(cudaMallocAsync((void **)&flags, 2 * B, s));
  if (!iters_used) LS_TRY(cudaMallocAsync((void **)&iters, sizeof(int32_t) * B, s));
  {
    int32_t *it_out = iters_used ? iters_used : iters;
    uint8_t *active = flags, *unsat = flags + B;
    LS_TRY(cudaMemsetAsync(c2v, 0, sizeof(double) * std::max<int64_t>(E, 1) * B, s));
    k_fill_u8<<<grid_for(B, 256), 256, 0, s>>>(active, B, 1);
    k_fill_u8<<<grid_for(B, 256), 256, 0, s>>>(unsat, B, 0);
    k_fill_i32<<<grid_for(B, 256), 256, 0, s>>>(it_out, B, num_iter);
    dim3 tgrid((unsigned)((n + 31) / 32), (unsigned)((B + 31) / 32)), tblk(32, 8);
    k_ex_init<T><<<tgrid, tblk, 0, s>>>(llr, B, n, chan, total);
    const int bt = 128;
    const unsigned gx = (unsigned)((B + bt - 1) / bt);
    dim3 gc(gx, (unsigned)std::min<int64_t>(m, 65535)), gv(gx, (unsigned)std::min<int64_t>(n, 65535));
    const int is_f32 = sizeof(T) == 4;
    const double alpha = variant == LS_SCALED_MIN_SUM ? scale : 1.0;
    for (int it = 0; it < num_iter; ++it) {
      const int first_f32 = is_f32 && it == 0;
      if (variant == LS_SUM_PRODUCT)
        k_ex_check<T, LS_SUM_PRODUCT><<<gc, bt, 0, s>>>(g->cptr, g->cvar, m, B, total, c2v, active, first_f32, alpha);
      else
        k_ex_check<T, LS_MIN_SUM><<<gc, bt, 0, s>>>(g->cptr, g->cvar, m, B, total, c2v, active, first_f32, alpha);
      k_ex_var<T><<<gv, bt, 0, s>>>(g->vptr, g->vedge, n, B, chan, total, c2v, active);
      if (early_stop) {
        k_ex_syndrome<T><<<gc, bt, 0, s>>>(g->cptr, g->cvar, m, B, total, active, unsat);
        k_ex_freeze<<<grid_for(B, 256), 256, 0, s>>>(B, active, unsat, it_out, it);
      }
    }
    k_ex_output<T><<<tgrid, tblk, 0, s>>>(total, B, n, out, hard);
  }
  e = cudaGetLastError();
fail_:
  if (chan) cudaFreeAsync(chan, s);
  if (total) cudaFreeAsync(total, s);
  if (c2v) cudaFreeAsync(c2v, s);
  if (flags) cudaFreeAsync(flags, s);
  if (iters) cudaFreeAsync(iters, s);
#undef LS_TRY
  return e == cudaSuccess ? LS_OK : cuda_status(e, "ls_bp_decode");
}

}  // namespace lsb

using namespace lsb;

extern "C" {

int ls_graph_create(int64_t n, int64_t m, const int64_t *cptr, const int64_t *cvar, ls_graph **out) {
  if (!out || !cptr || (m && !cvar)) return fail(LS_EINVAL, "ls_graph_create: null argument");
  if (n < 1 || m < 0) return fail(LS_EINVAL, "ls_graph_create: bad dimensions");
  const int64_t E = cptr[m];
  std::vector<int32_t> hc(m + 1), hv(E), vp(n + 1, 0), ve(E);
  int max_c = 0, max_v = 0;
  for (int64_t c = 0; c <= m; ++c) hc[c] = (int32_t)cptr[c];
  for (int64_t c = 0; c < m; ++c) {
    if (cptr[c + 1] < cptr[c]) return fail(LS_EINVAL, "ls_graph_create: cptr not monotone");
    max_c = std::max<int>(max_c, (int)(cptr[c + 1] - cptr[c]));
    for (int64_t e = cptr[c]; e < cptr[c + 1]; ++e) {
      if (cvar[e] < 0 || cvar[e] >= n) return fail(LS_EINVAL, "variable index out of range");
      if (e > cptr[c] && cvar[e] <= cvar[e - 1]) return fail(LS_EINVAL, "ls_graph_create: variables must ascend per check");
      hv[e] = (int32_t)cvar[e];
      vp[cvar[e] + 1]++;
    }
  }
  for (int64_t v = 0; v < n; ++v) {
    max_v = std::max<int>(max_v, vp[v + 1]);
    vp[v + 1] += vp[v];
  }
  {
    std::vector<int32_t> fill(vp.begin(), vp.end() - 1);
    for (int64_t e = 0; e < E; ++e) ve[fill[hv[e]]++] = (int32_t)e;  // ascending check order
  }
  ls_graph *g = new ls_graph();
  g->n = n; g->m = m; g->E = E; g->max_cdeg = max_c; g->max_vdeg = max_v;
  cudaError_t e = cudaSuccess;
  if ((e = cudaMalloc(&g->cptr, sizeof(int32_t) * (m + 1))) != cudaSuccess ||
      (e = cudaMalloc(&g->cvar, sizeof(int32_t) * std::max<int64_t>(E, 1))) != cudaSuccess ||
      (e = cudaMalloc(&g->vptr, sizeof(int32_t) * (n + 1))) != cudaSuccess ||
      (e = cudaMalloc(&g->vedge, sizeof(int32_t) * std::max<int64_t>(E, 1))) != cudaSuccess ||
      (e = cudaMemcpy(g->cptr, hc.data(), sizeof(int32_t) * (m + 1), cudaMemcpyHostToDevice)) != cudaSuccess ||
      (E && (e = cudaMemcpy(g->cvar, hv.data(), sizeof(int32_t) * E, cudaMemcpyHostToDevice)) != cudaSuccess) ||
      (e = cudaMemcpy(g->vptr, vp.data(), sizeof(int32_t) * (n + 1), cudaMemcpyHostToDevice)) != cudaSuccess ||
      (E && (e = cudaMemcpy(g->vedge, ve.data(), sizeof(int32_t) * E, cudaMemcpyHostToDevice)) != cudaSuccess)) {
    ls_graph_destroy(g);
    return cuda_status(e, "ls_graph_create");
  }
  *out = g;
  return LS_OK;
}

int ls_graph_from_code(const ls_code *code, ls_graph **out) {
  if (!code || !out) return fail(LS_EINVAL, "ls_graph_from_code: null argument");
  const QcParams &P = code->p;
  const int Z = P.z;
  // CN r*Z+i <-> VN c*Z+(i+s)%Z (ldpc.py:282-295); variables ascend per check
  std::vector<std::vector<int64_t>> rows(P.m_full);
  for (int e = 0; e < P.nnz; ++e) {
    const int r = code->entries[3 * e], c = code->entries[3 * e + 1], s = P.s[e];
    for (int i = 0; i < Z; ++i) rows[(int64_t)r * Z + i].push_back((int64_t)c * Z + (i + s) % Z);
  }
  std::vector<int64_t> cptr(P.m_full + 1, 0), cvar;
  cvar.reserve((size_t)P.nnz * Z);
  for (int64_t c = 0; c < P.m_full; ++c) {
    std::sort(rows[c].begin(), rows[c].end());
    cvar.insert(cvar.end(), rows[c].begin(), rows[c].end());
    cptr[c + 1] = (int64_t)cvar.size();
  }
  return ls_graph_create(P.n_full, P.m_full, cptr.data(), cvar.data(), out);
}

int ls_graph_destroy(ls_graph *g) {
  if (!g) return LS_OK;
  cudaFree(g->cptr);
  cudaFree(g->cvar);
  cudaFree(g->vptr);
  cudaFree(g->vedge);
  delete g;
  return LS_OK;
}

int ls_bp_decode(const ls_graph *g, const void *llr, int is_f64, int64_t batch, int num_iter, int variant,
                 double scale, int early_stop, void *llr_out, uint8_t *hard, int32_t *iters_used,
                 void *stream) {
  if (!g) return fail(LS_EINVAL, "ls_bp_decode: null graph");
  if (variant < 0 || variant > 2) return fail(LS_EINVAL, "unknown BP variant");
  if (num_iter < 1) return fail(LS_EINVAL, "num_iter must be >= 1");
  if (batch < 0) return fail(LS_EINVAL, "ls_bp_decode: negative batch");
  if (!batch) return LS_OK;
  cudaStream_t s = as_stream(stream);
  // rows are independent: bound the [E, B] f64 workspace to ~8 GB by
  // decoding in row chunks (same results as one call)
  const int64_t per_row = 8 * std::max<int64_t>(g->E, 1) + 16 * g->n + 16;
  const int64_t chunk = std::max<int64_t>(32, (8LL << 30) / per_row);
  const size_t esz = is_f64 ? 8 : 4;
  for (int64_t b0 = 0; b0 < batch; b0 += chunk) {
    const int64_t nb = std::min(chunk, batch - b0);
    const char *in = (const char *)llr + (size_t)b0 * g->n * esz;
    char *out = llr_out ? (char *)llr_out + (size_t)b0 * g->n * esz : nullptr;
    uint8_t *hd = hard ? hard + (size_t)b0 * g->n : nullptr;
    int32_t *it = iters_used ? iters_used + b0 : nullptr;
    const int rc = is_f64 ? run_exact<double>(g, (const double *)in, nb, num_iter, variant, scale, early_stop,
                                              (double *)out, hd, it, s)
                          : run_exact<float>(g, (const float *)in, nb, num_iter, variant, scale, early_stop,
                                             (float *)out, hd, it, s);
    if (rc != LS_OK) return rc;
  }
  return LS_OK;
}

}  // extern "C"
