// FAST-mode QC sum-product decoder (ldpc.py:139-143 check update) -- the
// reference's default BP variant on the on-chip flooding schedule.
//
// Unlike min-sum, the sum-product check output of every edge depends on that
// edge's own input, so the check-node state does not compress to a few words
// per check: every check-to-variable message is kept, as fp16, in shared
// memory, edge-block-major (c2v[e][i] = message of circulant entry e, check
// lane i).  That also removes the VN-phase barriers of the min-sum kernels:
// the variable update is a pure gather, total[c][j] = chan + sum over the
// column's entries of c2v[e][(j - s_e) mod Z].
//   CN phase (thread = lane i, row slot h): v2c = total - c2v_old,
//            phi(x) = -log(tanh(x/2)) (ex2/rcp/lg2 MUFU, fp32), S = sum phi,
//            c2v_new = sign * clip(phi(max(S - phi_e, 1e-12)), 0, 30)
//   VN phase (thread = lane j, column slot): gather + clip +-40
// Shared memory: E_live*Z halves of messages + NCOL*Z halves of posteriors
// (207 KB for BG1, Z=384, 24 live rows).  Channel LLRs are re-read from the
// rate-matched input (L2-resident) in each VN phase.
#pragma once

#include <cuda_fp16.h>

#include "bp_fast_qc.cuh"

namespace lsb {

template <class G, int Z, int R, int SPLIT>
struct QcShapeSP {
  static constexpr int NT1 = ((Z + 31) / 32) * 32;
  static constexpr int NT = NT1 * SPLIT;
  static constexpr int NCOL = G::KB + (R > 4 ? R : 4);
  static constexpr int NE = G::row_start[R];  // live base entries
  static constexpr size_t SMEM = 2ull * ((size_t)NE * Z + (size_t)NCOL * Z);
  static constexpr int MINB = NT >= 384 ? 1 : (384 / NT);
};

// phi(x) = -log(tanh(x / 2)) on the reference's clip range [1e-12, 40]
// (3 MUFU: ex2, rcp, lg2; branch-free).  phi(x) = ln((1 + u) / (1 - u)) with
// u = e^-x; for small x the denominator 1 - u comes from its Taylor series
// (no cancellation).
__device__ __forceinline__ float sp_phi(float x) {
  x = fminf(fmaxf(x, 1e-12f), 40.0f);
  const float u = __expf(-x);
  const float series = x * fmaf(x, fmaf(x, fmaf(x, -1.0f / 24.0f, 1.0f / 6.0f), -0.5f), 1.0f);
  const float om = x < 0.0625f ? series : 1.0f - u;
  return __logf(__fdividef(1.0f + u, om));
}

template <class G, int Z, int E>
__device__ __forceinline__ unsigned vn_off2(unsigned i2) {  // byte offset of (c, (i+s)%Z), 2-byte elements
  constexpr unsigned S2 = 2u * (unsigned)(G::shift[E] % Z);
  constexpr unsigned CB = 2u * (unsigned)Z * (unsigned)G::col[E];
  if constexpr (S2 == 0) return CB + i2;
  return CB + min(i2 + S2, i2 + (S2 - 2u * (unsigned)Z));
}

template <class G, int Z, int R, int SPLIT>
__global__ void __launch_bounds__(QcShapeSP<G, Z, R, SPLIT>::NT, QcShapeSP<G, Z, R, SPLIT>::MINB)
    k_qc_sp(const QcChanParams P, const float *__restrict__ llr, int num_iter, int early_stop,
            uint8_t *__restrict__ hard_k, float *__restrict__ llr_out, int32_t *__restrict__ iters_used,
            const uint8_t *__restrict__ ref, unsigned long long *__restrict__ counts) {
  using S = QcShapeSP<G, Z, R, SPLIT>;
  extern __shared__ __half smh[];
  __half *c2v = smh;                        // [NE][Z]
  __half *tot = smh + (size_t)S::NE * Z;    // [NCOL][Z]
  char *const totb = reinterpret_cast<char *>(tot);
  const int t = threadIdx.x;
  const int h = t / S::NT1;
  const int i = t - h * S::NT1;
  const bool lane = i < Z;
  const int64_t b = blockIdx.x;
  const float *row = llr + b * (int64_t)P.n;

  for (int v = t; v < S::NCOL * Z; v += S::NT) tot[v] = __float2half_rn(chan_value(P, row, v));
  for (int q = t; q < S::NE * Z; q += S::NT) c2v[q] = __float2half_rn(0.0f);
  __syncthreads();

  int used = num_iter;
  for (int it = 0; it < num_iter; ++it) {
    // ------------------------------------------------ check-node phase
    uint32_t synx = 0;
    if (lane) {
      sfor<0, SPLIT>([&](auto hc) {
        constexpr int H = decltype(hc)::value;
        if (h != H) return;
        const unsigned i2 = 2u * (tid_volatile() - H * S::NT1);
        const int il = (int)(i2 >> 1);
        sfor<0, (R + SPLIT - 1) / SPLIT>([&](auto jc) {
          constexpr int r = decltype(jc)::value * SPLIT + H;
          if constexpr (r < R) {
            constexpr int e0 = G::row_start[r], e1 = G::row_start[r + 1], d = e1 - e0;
            float ph[d];
            uint32_t sg = 0, hs = 0;
            float ssum = 0.0f;
            sfor<e0, e1>([&](auto ec) {
              constexpr int e = decltype(ec)::value;
              constexpr int p = e - e0;
              const __half th = *reinterpret_cast<const __half *>(totb + vn_off2<G, Z, e>(i2));
              hs ^= (uint32_t)__half_as_ushort(th);
              const float x = __half2float(th) - __half2float(c2v[e * Z + il]);
              sg |= (__float_as_uint(x) >> 31) << p;
              ph[p] = sp_phi(fabsf(x));
              ssum += ph[p];
            });
            const uint32_t par = __popc(sg) & 1u;
            sfor<e0, e1>([&](auto ec) {
              constexpr int e = decltype(ec)::value;
              constexpr int p = e - e0;
              const float m = fminf(sp_phi(fmaxf(ssum - ph[p], 1e-12f)), 30.0f);
              const bool neg = (par ^ (sg >> p)) & 1u;
              c2v[e * Z + il] = __float2half_rn(neg ? -m : m);
            });
            synx |= hs;
          }
        });
      });
    }
    if (early_stop && it > 0) {
      if (!__syncthreads_or(lane && ((synx >> 15) & 1u))) {  // fp16 sign bit
        used = it;
        break;
      }
    } else {
      __syncthreads();
    }
    // ------------------------------------------------ variable-node phase (gather)
    if (lane) {
      sfor<0, SPLIT>([&](auto hc) {
        constexpr int H = decltype(hc)::value;
        if (h != H) return;
        const int j = (int)tid_volatile() - H * S::NT1;
        sfor<0, (S::NCOL + SPLIT - 1) / SPLIT>([&](auto cc) {
          constexpr int c = decltype(cc)::value * SPLIT + H;
          if constexpr (c < S::NCOL) {
            float sum = chan_value(P, row, c * Z + j);
            constexpr int q0 = G::col_start[c], q1 = G::col_start[c + 1];
            sfor<q0, q1>([&](auto qc) {
              constexpr int e = G::col_entry[decltype(qc)::value];
              if constexpr (G::row[e] < R) {
                constexpr unsigned ZS = (unsigned)(Z - G::shift[e] % Z);  // (j - s) mod Z = (j + Z - s) mod Z
                const unsigned a = (unsigned)j + ZS;
                const unsigned src = min(a, a - (unsigned)Z);
                sum += __half2float(c2v[e * Z + src]);
              }
            });
            tot[c * Z + j] = __float2half_rn(fminf(fmaxf(sum, -40.0f), 40.0f));
          }
        });
      });
    }
    __syncthreads();
  }

  // ------------------------------------------------ outputs
  if (iters_used && t == 0) iters_used[b] = used;
  if (llr_out) {
    float *o = llr_out + b * (int64_t)P.n_full;
    for (int v = t; v < P.n_full; v += S::NT)
      o[v] = v < S::NCOL * Z ? -__half2float(tot[v]) : -chan_value(P, row, v);
  }
  unsigned err = 0;
  for (int v = t; v < P.k; v += S::NT) {
    const uint8_t hd = (-__half2float(tot[v])) > 0.0f;
    if (hard_k) hard_k[b * (int64_t)P.k + v] = hd;
    if (ref) err += (hd != ref[b * (int64_t)P.k + v]);
  }
  if (ref && counts) {
    __shared__ unsigned red[S::NT / 32];
#pragma unroll
    for (int o = 16; o; o >>= 1) err += __shfl_xor_sync(0xffffffffu, err, o);
    if ((t & 31) == 0) red[t >> 5] = err;
    __syncthreads();
    if (t == 0) {
      unsigned long long tt = 0;
      for (int w = 0; w < S::NT / 32; ++w) tt += red[w];
      if (tt) {
        atomicAdd(&counts[0], tt);
        atomicAdd(&counts[1], 1ULL);
      }
    }
  }
}

template <class G, int Z, int R, int SPLIT>
int launch_qc_sp(const QcChanParams &P, const float *llr, int64_t B, int num_iter, float alpha, int early_stop,
                 uint8_t *hard_k, float *llr_out, int32_t *iters_used, const uint8_t *ref,
                 unsigned long long *counts, cudaStream_t s) {
  (void)alpha;
  using S = QcShapeSP<G, Z, R, SPLIT>;
  static_assert(S::SMEM <= 227 * 1024, "sum-product messages do not fit in shared memory");
  auto kern = k_qc_sp<G, Z, R, SPLIT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMEM);
  if (e != cudaSuccess) return cuda_status(e, "ls_qc_decode(smem attr)");
  for (int64_t b0 = 0; b0 < B; b0 += 0x7fffffff) {
    const int64_t nb = B - b0 < 0x7fffffff ? B - b0 : 0x7fffffff;
    kern<<<(unsigned)nb, S::NT, S::SMEM, s>>>(P, llr + b0 * P.n, num_iter, early_stop,
                                              hard_k ? hard_k + b0 * P.k : nullptr,
                                              llr_out ? llr_out + b0 * P.n_full : nullptr,
                                              iters_used ? iters_used + b0 : nullptr,
                                              ref ? ref + b0 * P.k : nullptr, counts);
  }
  e = cudaGetLastError();
  return e == cudaSuccess ? LS_OK : cuda_status(e, "ls_qc_decode");
}

}  // namespace lsb
