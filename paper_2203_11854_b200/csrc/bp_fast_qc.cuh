// Specialised FAST-mode QC decoder (F2): base graph, lifting size Z and the
// number of processed rows R are compile-time, so every shift, column base
// and loop bound is an immediate and the check-node state of the R rows stays
// in registers.  Included by the bp_fast_inst_*.cu instantiation units.
//
// Same schedule and numerics as the runtime-Z kernel in bp_fast.cu:
//   CN phase: v2c = total[v] - c2v_old;  compressed (min1, min2, argmin,
//             sign bits) per check; syndrome of `total` on the side;
//   VN phase: total = chan + sum c2v_new (row by row, barrier between rows),
//             clip +-40.
// R < m_b drops the "dead" extension rows whose degree-1 parity VN is never
// transmitted: they only ever send signed zeros (up to
// the |c2v| > 40 corner), so skipping them is a fast-mode optimisation,
// validated statistically (tests/test_gpu_parity.py).
#pragma once

#include <type_traits>

#include "common.cuh"

namespace lsb {

template <int B_, int E_, class F>
__device__ __forceinline__ void sfor(F &&f) {
  if constexpr (B_ < E_) {
    f(std::integral_constant<int, B_>{});
    sfor<B_ + 1, E_>(f);
  }
}

struct QcChanParams {
  int z, k, n, k_full, n_full, l1, buflen;
};

__device__ __forceinline__ float chan_value(const QcChanParams &P, const float *__restrict__ row, int v) {
  if (v >= P.k && v < P.k_full) return 40.0f;  // filler: mother -40 (ldpc.py:344)
  if (v < 2 * P.z) return -0.0f;               // punctured: mother +0.0
  const int pos = v < P.k ? v - 2 * P.z : P.l1 + (v - P.k_full);
  float acc = 0.0f;
  for (int j = pos; j < P.n; j += P.buflen) acc += __ldg(row + j);
  return -acc;
}

// Thread layout: SPLIT threads per circulant lane.  Thread t serves lane
// t % NT1 and owns the rows r with r % SPLIT == t / NT1 ("slot" h), so the
// check-node state per thread is ceil(R / SPLIT) rows and a CTA has
// SPLIT * NT1 threads (more warps per SM for the same codeword).  In the VN
// phase slot h accumulates its rows into its own array (slot 0 into `tot`),
// one row per slot per barrier step, and the slots are summed at the end.
template <class G, int Z, int R, int SPLIT>
struct QcShape {
  static constexpr int NT1 = ((Z + 31) / 32) * 32;      // threads per slot
  static constexpr int NT = NT1 * SPLIT;                // threads per codeword
  static constexpr int NCOL = G::KB + (R > 4 ? R : 4);  // columns touched by rows < R
  static constexpr int NV = NCOL * Z;                   // posteriors in smem
  static constexpr int NR = (R + SPLIT - 1) / SPLIT;    // rows per thread
  static constexpr size_t ARR = sizeof(float) * (size_t)NV;
  static constexpr bool CHN_SMEM = (SPLIT + 1) * ARR <= 225 * 1024;  // cache channel LLRs
  static constexpr size_t SMEM = (SPLIT + (CHN_SMEM ? 1 : 0)) * ARR;
  static constexpr int MINB = NT >= 384 ? 1 : (384 / NT);
};

// byte offset of VN (c, (i + s) mod Z) relative to the array base, for lane
// byte offset i4 = 4 i: min over the unwrapped / wrapped candidates (the
// wrapped one underflows to a huge unsigned value when i + s < Z)
template <class G, int Z, int E>
__device__ __forceinline__ unsigned vn_off(unsigned i4) {
  constexpr unsigned S4 = 4u * (unsigned)(G::shift[E] % Z);
  constexpr unsigned CB = 4u * (unsigned)Z * (unsigned)G::col[E];
  if constexpr (S4 == 0) return CB + i4;
  return CB + min(i4 + S4, i4 + (S4 - 4u * (unsigned)Z));
}

// %tid.x re-read through volatile asm: the compiler would otherwise hoist all
// R*deg loop-invariant VN addresses out of the iteration loop and spill them.
__device__ __forceinline__ unsigned tid_volatile() {
  unsigned t;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(t));
  return t;
}

template <class G, int Z, int R, int SPLIT>
__global__ void __launch_bounds__(QcShape<G, Z, R, SPLIT>::NT, QcShape<G, Z, R, SPLIT>::MINB)
    k_qc_fast2(const QcChanParams P, const float *__restrict__ llr, int num_iter, float alpha, int early_stop,
               uint8_t *__restrict__ hard_k, float *__restrict__ llr_out, int32_t *__restrict__ iters_used,
               const uint8_t *__restrict__ ref, unsigned long long *__restrict__ counts) {
  using S = QcShape<G, Z, R, SPLIT>;
  extern __shared__ float sm[];
  float *tot = sm;                          // slot-0 accumulator / posterior
  float *chn = sm + SPLIT * S::NV;          // channel LLRs (if cached)
  const int t = threadIdx.x;
  const int h = t / S::NT1;                 // row slot (warp-uniform)
  const int i = t - h * S::NT1;             // circulant lane
  const bool lane = i < Z;
  char *const base = reinterpret_cast<char *>(sm);
  const int64_t b = blockIdx.x;
  const float *row = llr + b * (int64_t)P.n;

  for (int v = t; v < S::NV; v += S::NT) {
    const float ch = chan_value(P, row, v);
    if constexpr (S::CHN_SMEM) chn[v] = ch;
    tot[v] = ch;
  }
  float m1[S::NR], m2[S::NR];
  uint32_t pk[S::NR];
#pragma unroll
  for (int j = 0; j < S::NR; ++j) {
    m1[j] = 0.0f;
    m2[j] = 0.0f;
    pk[j] = 0u;
  }
  __syncthreads();

  int used = num_iter;
  for (int it = 0; it < num_iter; ++it) {
    // ------------------------------------------------ check-node phase
    uint32_t synx = 0;
    if (lane) {
      sfor<0, SPLIT>([&](auto hc) {
        constexpr int H = decltype(hc)::value;
        if (h != H) return;
        const unsigned i4 = 4u * tid_volatile() - 4u * H * S::NT1;
        sfor<0, S::NR>([&](auto jc) {
          constexpr int j = decltype(jc)::value;
          constexpr int r = j * SPLIT + H;
          if constexpr (r < R) {
            constexpr int e0 = G::row_start[r], e1 = G::row_start[r + 1], d = e1 - e0;
            const float o1 = m1[j], o2 = m2[j];
            const uint32_t opk = pk[j];
            const uint32_t oidx = opk >> 27;
            float n1 = INFINITY, n2 = INFINITY;
            uint32_t idx = 0, sg = 0, hs = 0;
            sfor<e0, e1>([&](auto ec) {
              constexpr int e = decltype(ec)::value;
              constexpr int p = e - e0;
              const float tv = *reinterpret_cast<const float *>(base + vn_off<G, Z, e>(i4));
              hs ^= __float_as_uint(tv);
              const float mag = (oidx == (uint32_t)p) ? o2 : o1;
              const float cold = __uint_as_float(__float_as_uint(mag) | ((opk << (31 - p)) & 0x80000000u));
              const float x = tv - cold;
              const float a = fabsf(x);
              idx = a < n1 ? (uint32_t)p : idx;
              n2 = fminf(n2, fmaxf(n1, a));
              n1 = fminf(n1, a);
              sg |= (__float_as_uint(x) >> 31) << p;
            });
            const uint32_t par = __popc(sg) & 1u;
            const uint32_t sgx = sg ^ ((0u - par) & ((1u << d) - 1u));
            m1[j] = alpha * n1;
            m2[j] = alpha * n2;
            pk[j] = (idx << 27) | sgx;
            synx |= hs;
          }
        });
      });
    }
    if (early_stop && it > 0) {
      // syndrome of the posterior left by iteration `it` (ldpc.py:155-160)
      if (!__syncthreads_or(lane && (synx >> 31))) {
        used = it;
        break;
      }
    } else {
      __syncthreads();
    }
    // ------------------------------------------------ variable-node phase
    for (int v = t; v < S::NV; v += S::NT) {
      float ch;
      if constexpr (S::CHN_SMEM) ch = chn[v];
      else ch = chan_value(P, row, v);
      tot[v] = ch;
#pragma unroll
      for (int q = 1; q < SPLIT; ++q) tot[q * S::NV + v] = 0.0f;
    }
    __syncthreads();
    sfor<0, S::NR>([&](auto jc) {
      constexpr int j = decltype(jc)::value;
      if (lane) {
        sfor<0, SPLIT>([&](auto hc) {
          constexpr int H = decltype(hc)::value;
          constexpr int r = j * SPLIT + H;
          if constexpr (r < R) {
            if (h != H) return;
            constexpr int e0 = G::row_start[r], e1 = G::row_start[r + 1];
            // the min-based wrap in vn_off needs the pure lane offset; the
            // slot's accumulator array is added to the base pointer instead
            const unsigned i4 = 4u * tid_volatile() - 4u * H * S::NT1;
            char *const arr = base + 4u * H * S::NV;
            const float o1 = m1[j], o2 = m2[j];
            const uint32_t opk = pk[j];
            const uint32_t oidx = opk >> 27;
            sfor<e0, e1>([&](auto ec) {
              constexpr int e = decltype(ec)::value;
              constexpr int p = e - e0;
              float *tp = reinterpret_cast<float *>(arr + vn_off<G, Z, e>(i4));
              const float mag = (oidx == (uint32_t)p) ? o2 : o1;
              const float cnew = __uint_as_float(__float_as_uint(mag) | ((opk << (31 - p)) & 0x80000000u));
              *tp = *tp + cnew;
            });
          }
        });
      }
      __syncthreads();
    });
    for (int v = t; v < S::NV; v += S::NT) {
      float acc = tot[v];
#pragma unroll
      for (int q = 1; q < SPLIT; ++q) acc += tot[q * S::NV + v];
      tot[v] = fminf(fmaxf(acc, -40.0f), 40.0f);
    }
    __syncthreads();
  }

  // ------------------------------------------------ outputs
  if (iters_used && t == 0) iters_used[b] = used;
  if (llr_out) {
    float *o = llr_out + b * (int64_t)P.n_full;
    for (int v = t; v < P.n_full; v += S::NT) o[v] = v < S::NV ? -tot[v] : -chan_value(P, row, v);
  }
  unsigned err = 0;
  for (int v = t; v < P.k; v += S::NT) {
    const uint8_t hd = (-tot[v]) > 0.0f;
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
#pragma unroll
      for (int w = 0; w < S::NT / 32; ++w) tt += red[w];
      if (tt) {
        atomicAdd(&counts[0], tt);
        atomicAdd(&counts[1], 1ULL);
      }
    }
  }
}

using QcLauncher = int (*)(const QcChanParams &, const float *, int64_t, int, float, int, uint8_t *, float *,
                           int32_t *, const uint8_t *, unsigned long long *, cudaStream_t);

template <class G, int Z, int R, int SPLIT>
int launch_qc_fast2(const QcChanParams &P, const float *llr, int64_t B, int num_iter, float alpha, int early_stop,
                    uint8_t *hard_k, float *llr_out, int32_t *iters_used, const uint8_t *ref,
                    unsigned long long *counts, cudaStream_t s) {
  using S = QcShape<G, Z, R, SPLIT>;
  auto kern = k_qc_fast2<G, Z, R, SPLIT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMEM);
  if (e != cudaSuccess) return cuda_status(e, "ls_qc_decode(smem attr)");
  for (int64_t b0 = 0; b0 < B; b0 += 0x7fffffff) {
    const int64_t nb = B - b0 < 0x7fffffff ? B - b0 : 0x7fffffff;
    kern<<<(unsigned)nb, S::NT, S::SMEM, s>>>(P, llr + b0 * P.n, num_iter, alpha, early_stop,
                                              hard_k ? hard_k + b0 * P.k : nullptr,
                                              llr_out ? llr_out + b0 * P.n_full : nullptr,
                                              iters_used ? iters_used + b0 : nullptr, ref ? ref + b0 * P.k : nullptr,
                                              counts);
  }
  e = cudaGetLastError();
  return e == cudaSuccess ? LS_OK : cuda_status(e, "ls_qc_decode");
}

// registry entry: (bg, Z, R) -> launcher, defined by the instantiation units
struct QcKernelEntry {
  int bg, z, r, prec;  // prec: 0 fp32, 1 fp16x2
  QcLauncher fn;
};

}  // namespace lsb
