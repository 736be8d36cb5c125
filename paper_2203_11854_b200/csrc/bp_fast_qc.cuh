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

template <class G, int Z, int R>
struct QcShape {
  static constexpr int NT = ((Z + 31) / 32) * 32;       // threads per codeword
  static constexpr int NCOL = G::KB + (R > 4 ? R : 4);  // columns touched by rows < R
  static constexpr size_t SMEM = 2ull * sizeof(float) * NCOL * Z;
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

// lane byte offset re-read from %tid.x through volatile asm: the compiler
// would otherwise hoist all R*deg loop-invariant VN addresses out of the
// iteration loop and spill them.
__device__ __forceinline__ unsigned lane_off4() {
  unsigned t;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(t));
  return 4u * t;
}

template <class G, int Z, int R>
__global__ void __launch_bounds__(QcShape<G, Z, R>::NT, QcShape<G, Z, R>::MINB)
    k_qc_fast2(const QcChanParams P, const float *__restrict__ llr, int num_iter, float alpha, int early_stop,
               uint8_t *__restrict__ hard_k, float *__restrict__ llr_out, int32_t *__restrict__ iters_used,
               const uint8_t *__restrict__ ref, unsigned long long *__restrict__ counts) {
  using S = QcShape<G, Z, R>;
  extern __shared__ float sm[];
  float *tot = sm;
  float *chn = sm + S::NCOL * Z;
  const int i = threadIdx.x;
  const bool lane = i < Z;
  char *tb = reinterpret_cast<char *>(tot);
  const int64_t b = blockIdx.x;
  const float *row = llr + b * (int64_t)P.n;

  if (lane) {
#pragma unroll 4
    for (int c = 0; c < S::NCOL; ++c) {
      const float ch = chan_value(P, row, c * Z + i);
      chn[c * Z + i] = ch;
      tot[c * Z + i] = ch;
    }
  }
  float m1[R], m2[R];
  uint32_t pk[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    m1[r] = 0.0f;
    m2[r] = 0.0f;
    pk[r] = 0u;
  }
  __syncthreads();

  int used = num_iter;
  for (int it = 0; it < num_iter; ++it) {
    uint32_t synx = 0;
    if (lane) {
      const unsigned i4 = lane_off4();
      sfor<0, R>([&](auto rc) {
        constexpr int r = decltype(rc)::value;
        constexpr int e0 = G::row_start[r], e1 = G::row_start[r + 1], d = e1 - e0;
        const float o1 = m1[r], o2 = m2[r];
        const uint32_t opk = pk[r];
        const uint32_t oidx = opk >> 27;
        float n1 = INFINITY, n2 = INFINITY;
        uint32_t idx = 0, sg = 0, hs = 0;
        sfor<e0, e1>([&](auto ec) {
          constexpr int e = decltype(ec)::value;
          constexpr int p = e - e0;
          const float t = *reinterpret_cast<const float *>(tb + vn_off<G, Z, e>(i4));
          hs ^= __float_as_uint(t);
          const float mag = (oidx == (uint32_t)p) ? o2 : o1;
          const float cold = __uint_as_float(__float_as_uint(mag) | ((opk << (31 - p)) & 0x80000000u));
          const float x = t - cold;
          const float a = fabsf(x);
          idx = a < n1 ? (uint32_t)p : idx;
          n2 = fminf(n2, fmaxf(n1, a));
          n1 = fminf(n1, a);
          sg |= (__float_as_uint(x) >> 31) << p;
        });
        const uint32_t par = __popc(sg) & 1u;
        const uint32_t sgx = sg ^ ((0u - par) & ((1u << d) - 1u));
        m1[r] = alpha * n1;
        m2[r] = alpha * n2;
        pk[r] = (idx << 27) | sgx;
        synx |= hs;
      });
    }
    if (early_stop && it > 0) {
      if (!__syncthreads_or(lane && (synx >> 31))) {
        used = it;
        break;
      }
    } else {
      __syncthreads();
    }
    if (lane) {
#pragma unroll 4
      for (int c = 0; c < S::NCOL; ++c) tot[c * Z + i] = chn[c * Z + i];
    }
    __syncthreads();
    sfor<0, R>([&](auto rc) {
      constexpr int r = decltype(rc)::value;
      constexpr int e0 = G::row_start[r], e1 = G::row_start[r + 1];
      if (lane) {
        const unsigned i4 = lane_off4();
        const float o1 = m1[r], o2 = m2[r];
        const uint32_t opk = pk[r];
        const uint32_t oidx = opk >> 27;
        sfor<e0, e1>([&](auto ec) {
          constexpr int e = decltype(ec)::value;
          constexpr int p = e - e0;
          float *tp = reinterpret_cast<float *>(tb + vn_off<G, Z, e>(i4));
          const float mag = (oidx == (uint32_t)p) ? o2 : o1;
          const float cnew = __uint_as_float(__float_as_uint(mag) | ((opk << (31 - p)) & 0x80000000u));
          *tp = *tp + cnew;
        });
      }
      __syncthreads();
    });
    if (lane) {
#pragma unroll 4
      for (int c = 0; c < S::NCOL; ++c) tot[c * Z + i] = fminf(fmaxf(tot[c * Z + i], -40.0f), 40.0f);
    }
    __syncthreads();
  }

  if (iters_used && i == 0) iters_used[b] = used;
  if (llr_out) {
    float *o = llr_out + b * (int64_t)P.n_full;
    for (int v = i; v < P.n_full; v += S::NT) o[v] = v < S::NCOL * Z ? -tot[v] : -chan_value(P, row, v);
  }
  unsigned err = 0;
  for (int v = i; v < P.k; v += S::NT) {
    const uint8_t h = (-tot[v]) > 0.0f;
    if (hard_k) hard_k[b * (int64_t)P.k + v] = h;
    if (ref) err += (h != ref[b * (int64_t)P.k + v]);
  }
  if (ref && counts) {
    __shared__ unsigned red[S::NT / 32];
#pragma unroll
    for (int o = 16; o; o >>= 1) err += __shfl_xor_sync(0xffffffffu, err, o);
    if ((i & 31) == 0) red[i >> 5] = err;
    __syncthreads();
    if (i == 0) {
      unsigned long long t = 0;
#pragma unroll
      for (int w = 0; w < S::NT / 32; ++w) t += red[w];
      if (t) {
        atomicAdd(&counts[0], t);
        atomicAdd(&counts[1], 1ULL);
      }
    }
  }
}

using QcLauncher = int (*)(const QcChanParams &, const float *, int64_t, int, float, int, uint8_t *, float *,
                           int32_t *, const uint8_t *, unsigned long long *, cudaStream_t);

template <class G, int Z, int R>
int launch_qc_fast2(const QcChanParams &P, const float *llr, int64_t B, int num_iter, float alpha, int early_stop,
                    uint8_t *hard_k, float *llr_out, int32_t *iters_used, const uint8_t *ref,
                    unsigned long long *counts, cudaStream_t s) {
  using S = QcShape<G, Z, R>;
  auto kern = k_qc_fast2<G, Z, R>;
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
  int bg, z, r;
  QcLauncher fn;
};

}  // namespace lsb
