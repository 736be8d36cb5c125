// FAST-mode QC flooding BP decoder (ldpc.py:86-172 / ldpc5g_decode 354-365)
// fused with derate_match (ldpc.py:335-345), hard decision (core.py:102-104)
// and count_errors (core.py:93-99).
//
// Mapping: one CTA per codeword, thread i = circulant lane i (Z <= 384).
// Thread i owns check r*Z+i of every base row r.  Its check-node state stays
// in REGISTERS for the whole decode in compressed min-sum form: (min1, min2)
// and a word holding the argmin position and the outgoing sign bits
// (already XORed with the row parity).  The variable-node posteriors
// (`total`, fp32, n_b*Z values) live in shared memory; the channel LLRs are
// re-read from the rate-matched input (L2-resident after the first pass)
// when the posteriors are rebuilt each iteration.
//
// One iteration (flooding schedule, same as the reference):
//   CN phase  : every row r: v2c = total[v] - c2v_old, new (min1,min2,idx,signs)
//               -- also the syndrome of `total` (early stop of the previous
//               iteration is decided here, ldpc.py:155-160)
//   VN phase  : total = chan; for each row: total[v] += c2v_new; clip +-40
// The base-graph structure is compile-time (bg_tables.h) so all row/entry
// loops unroll and the state arrays stay in registers; the per-code shifts
// arrive as kernel parameters (constant bank).
#include <math.h>

#include <algorithm>
#include <type_traits>

#include "bp_fast_h2.cuh"
#include "bp_fast_qc.cuh"
#include "common.cuh"
#include "qc_instances.h"

namespace lsb {

// compile-time loop: f(std::integral_constant<int, I>) for I in [B, E)
template <int B_, int E_, class F>
__device__ __forceinline__ void static_for(F &&f) {
  if constexpr (B_ < E_) {
    f(std::integral_constant<int, B_>{});
    static_for<B_ + 1, E_>(f);
  }
}

// per-entry byte offsets into the posterior array: address of VN
// c*Z + (i+s)%Z is 4*i + (i < thr ? lo : hi)
struct QcFastParams {
  int z, k, n, k_full, n_full, l1, buflen;
  int nrows;  // base rows processed (dead extension rows pruned)
  int thr[kMaxNnz];
  int lo[kMaxNnz];
  int hi[kMaxNnz];
};

__device__ __forceinline__ float chan_of(const QcFastParams &P, const float *__restrict__ row, int v) {
  if (v >= P.k && v < P.k_full) return 40.0f;  // filler: mother -40 (ldpc.py:344)
  if (v < 2 * P.z) return -0.0f;               // punctured: mother +0.0
  const int pos = v < P.k ? v - 2 * P.z : P.l1 + (v - P.k_full);
  float acc = 0.0f;
  for (int j = pos; j < P.n; j += P.buflen) acc += __ldg(row + j);
  return -acc;
}

template <class G, int VARIANT>
__global__ void __launch_bounds__(384, 1)
    k_qc_fast(const QcFastParams P, const float *__restrict__ llr, int num_iter, float alpha, int early_stop,
              uint8_t *__restrict__ hard_k, float *__restrict__ llr_out, int32_t *__restrict__ iters_used,
              const uint8_t *__restrict__ ref, unsigned long long *__restrict__ counts) {
  extern __shared__ float tot[];  // [NB * Z]
  const int Z = P.z;
  const int i = threadIdx.x;
  const bool lane = i < Z;
  const int64_t b = blockIdx.x;
  const float *row = llr + b * (int64_t)P.n;
  char *tb = reinterpret_cast<char *>(tot) + 4 * i;  // lane-relative byte base

  float m1[G::MB], m2[G::MB];
  uint32_t pk[G::MB];
#pragma unroll
  for (int r = 0; r < G::MB; ++r) {
    m1[r] = 0.0f;
    m2[r] = 0.0f;
    pk[r] = 0u;
  }
  if (lane)
    for (int c = 0; c < G::NB; ++c) tot[c * Z + i] = chan_of(P, row, c * Z + i);
  __syncthreads();

  int used = num_iter;
  for (int it = 0; it < num_iter; ++it) {
    // ------------------------------------------------ check-node phase
    uint32_t synx = 0;
    if (lane) {
      static_for<0, G::MB>([&](auto rc) {
        constexpr int r = decltype(rc)::value;
        constexpr int e0 = G::row_start[r], e1 = G::row_start[r + 1];
        if (r >= P.nrows) return;
        const float o1 = m1[r], o2 = m2[r];
        const uint32_t opk = pk[r];
        const uint32_t oidx = opk & 31u;
        float n1 = INFINITY, n2 = INFINITY;
        uint32_t idx = 0, sg = 0, hs = 0;
#pragma unroll
        for (int e = e0; e < e1; ++e) {
          const int p = e - e0;
          const int off = i < P.thr[e] ? P.lo[e] : P.hi[e];
          const float t = *reinterpret_cast<const float *>(tb + off);
          hs ^= __float_as_uint(t);
          const float mag = (oidx == (uint32_t)p) ? o2 : o1;
          const float cold = __uint_as_float(__float_as_uint(mag) | ((opk << (26 - p)) & 0x80000000u));
          const float x = t - cold;
          const float a = fabsf(x);
          idx = a < n1 ? (uint32_t)p : idx;
          n2 = fminf(n2, fmaxf(n1, a));
          n1 = fminf(n1, a);
          sg |= (__float_as_uint(x) >> 31) << p;
        }
        const uint32_t par = __popc(sg) & 1u;
        const uint32_t sgx = sg ^ (par ? ((1u << (e1 - e0)) - 1u) : 0u);
        m1[r] = alpha * n1;
        m2[r] = alpha * n2;
        pk[r] = idx | (sgx << 5);
        synx |= hs;
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
    if (lane)
      for (int c = 0; c < G::NB; ++c) tot[c * Z + i] = chan_of(P, row, c * Z + i);
    __syncthreads();
    static_for<0, G::MB>([&](auto rc) {
      constexpr int r = decltype(rc)::value;
      if (r >= P.nrows) return;  // uniform: whole CTA skips the barrier
      if (lane) {
        constexpr int e0 = G::row_start[r], e1 = G::row_start[r + 1];
        const float o1 = m1[r], o2 = m2[r];
        const uint32_t opk = pk[r];
        const uint32_t oidx = opk & 31u;
#pragma unroll
        for (int e = e0; e < e1; ++e) {
          const int p = e - e0;
          const int off = i < P.thr[e] ? P.lo[e] : P.hi[e];
          float *tp = reinterpret_cast<float *>(tb + off);
          const float mag = (oidx == (uint32_t)p) ? o2 : o1;
          const float cnew = __uint_as_float(__float_as_uint(mag) | ((opk << (26 - p)) & 0x80000000u));
          *tp = *tp + cnew;
        }
      }
      __syncthreads();
    });
    if (lane)
      for (int c = 0; c < G::NB; ++c) tot[c * Z + i] = fminf(fmaxf(tot[c * Z + i], -40.0f), 40.0f);
    __syncthreads();
  }

  // ------------------------------------------------ outputs
  if (iters_used && i == 0) iters_used[b] = used;
  if (llr_out) {
    float *o = llr_out + b * (int64_t)P.n_full;
    for (int v = i; v < P.n_full; v += blockDim.x) o[v] = -tot[v];
  }
  unsigned err = 0;
  for (int v = i; v < P.k; v += blockDim.x) {
    const uint8_t h = (-tot[v]) > 0.0f;
    if (hard_k) hard_k[b * (int64_t)P.k + v] = h;
    if (ref) err += (h != ref[b * (int64_t)P.k + v]);
  }
  if (ref && counts) {
    __shared__ unsigned red[12];
    for (int o = 16; o; o >>= 1) err += __shfl_xor_sync(0xffffffffu, err, o);
    if ((i & 31) == 0) red[i >> 5] = err;
    __syncthreads();
    if (i == 0) {
      unsigned long long t = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
      if (t) {
        atomicAdd(&counts[0], t);
        atomicAdd(&counts[1], 1ULL);
      }
    }
  }
}

template <class G, int VARIANT>
static int launch_fast(const QcFastParams &FP, const float *llr, int64_t B, int num_iter, float alpha,
                       int early_stop, uint8_t *hard_k, float *llr_out, int32_t *iters_used, const uint8_t *ref,
                       unsigned long long *counts, cudaStream_t s) {
  const int threads = ((FP.z + 31) / 32) * 32;
  const size_t smem = sizeof(float) * (size_t)G::NB * FP.z;
  auto kern = k_qc_fast<G, VARIANT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return cuda_status(e, "ls_qc_decode(smem attr)");
  for (int64_t b0 = 0; b0 < B; b0 += 0x7fffffff) {
    const int64_t nb = std::min<int64_t>(B - b0, 0x7fffffff);
    kern<<<(unsigned)nb, threads, smem, s>>>(FP, llr + b0 * FP.n, num_iter, alpha, early_stop,
                                             hard_k ? hard_k + b0 * FP.k : nullptr,
                                             llr_out ? llr_out + b0 * FP.n_full : nullptr,
                                             iters_used ? iters_used + b0 : nullptr, ref ? ref + b0 * FP.k : nullptr,
                                             counts);
  }
  LS_CHECK_LAUNCH("ls_qc_decode");
  return LS_OK;
}

}  // namespace lsb

using namespace lsb;

namespace lsb {
#define LSB_QC_DECL(bg, z, r, sp, pr)                                                                   \
  int qc2_##pr##_##bg##_##z##_##r(const QcChanParams &, const float *, int64_t, int, float, int, uint8_t *, \
                                  float *, int32_t *, const uint8_t *, unsigned long long *, cudaStream_t);
LSB_QC_INSTANCES(LSB_QC_DECL)
#define LSB_QC_PREC_f32 0
#define LSB_QC_PREC_h2 1
#define LSB_QC_PREC_sp 2
#define LSB_QC_PREC_sp32 3
#define LSB_QC_ENTRY(bg, z, r, sp, pr) {bg, z, r, LSB_QC_PREC_##pr, &qc2_##pr##_##bg##_##z##_##r},
static const QcKernelEntry kQcKernels[] = {LSB_QC_INSTANCES(LSB_QC_ENTRY)};

typedef int (*QcRtFn)(const QcChanParams &, int, const uint16_t *, const int32_t *, const float *, int64_t, int,
                      float, int, uint8_t *, float *, int32_t *, const uint8_t *, unsigned long long *,
                      cudaStream_t);
#define LSB_QC_RT_DECL(bg, rb, sp)                                                                           \
  int qcrt_##bg##_##rb##_##sp(const QcChanParams &, int, const uint16_t *, const int32_t *, const float *, \
                              int64_t, int, float, int, uint8_t *, float *, int32_t *, const uint8_t *,    \
                              unsigned long long *, cudaStream_t);
LSB_QC_RT_INSTANCES(LSB_QC_RT_DECL)
struct QcRtEntry {
  int bg, rb, split;
  QcRtFn fn;
};
#define LSB_QC_RT_ENTRY(bg, rb, sp) {bg, rb, sp, &qcrt_##bg##_##rb##_##sp},
static const QcRtEntry kQcRtKernels[] = {LSB_QC_RT_INSTANCES(LSB_QC_RT_ENTRY)};

#define LSB_QC_SPRT_DECL(bg, rb, sp)                                                                           \
  int qcsprt_##bg##_##rb##_##sp(const QcChanParams &, int, const uint16_t *, const int32_t *, const float *, \
                                int64_t, int, float, int, uint8_t *, float *, int32_t *, const uint8_t *,    \
                                unsigned long long *, cudaStream_t);
LSB_QC_SPRT_INSTANCES(LSB_QC_SPRT_DECL)
#define LSB_QC_SPRT_ENTRY(bg, rb, sp) {bg, rb, sp, &qcsprt_##bg##_##rb##_##sp},
static const QcRtEntry kQcSpRtKernels[] = {LSB_QC_SPRT_INSTANCES(LSB_QC_SPRT_ENTRY)};

typedef int (*QcxFn)(const QcChanParams &, const float *, int64_t, int, double, int, int, uint8_t *, int, float *,
                     int32_t *, const uint8_t *, unsigned long long *, cudaStream_t);
#define LSB_QCX_DECL(bg, z, ntl)                                                                              \
  int qcx_##bg##_##z(const QcChanParams &, const float *, int64_t, int, double, int, int, uint8_t *, int, float *, \
                     int32_t *, const uint8_t *, unsigned long long *, cudaStream_t);                          \
  int qcf_##bg##_##z(const QcChanParams &, const float *, int64_t, int, double, int, int, uint8_t *, int, float *, \
                     int32_t *, const uint8_t *, unsigned long long *, cudaStream_t);
LSB_QCX_INSTANCES(LSB_QCX_DECL)
struct QcxEntry {
  int bg, z;
  QcxFn fn;   // f64 messages: exact
  QcxFn fn32; // f32 messages: fp32 full-graph fast mode
};
#define LSB_QCX_ENTRY(bg, z, ntl) {bg, z, &qcx_##bg##_##z, &qcf_##bg##_##z},
static const QcxEntry kQcxKernels[] = {LSB_QCX_INSTANCES(LSB_QCX_ENTRY)};

static const QcxEntry *find_qcx(const ls_code *code) {
  if (!code->std_shifts) return nullptr;
  for (const QcxEntry &k : kQcxKernels)
    if (k.bg == code->p.bg && k.z == code->p.z) return &k;
  return nullptr;
}

// runtime-geometry fp16x2 instance for (BG, Z, R): smallest row bound >= R,
// then the most threads per lane that fit 768 threads
template <size_t N>
static const QcRtEntry *pick_rt(const QcRtEntry (&table)[N], int bg, int z, int R) {
  const QcRtEntry *best = nullptr;
  const int nt1 = ((z + 31) / 32) * 32;
  for (const QcRtEntry &k : table) {
    if (k.bg != bg || k.rb < R || nt1 * k.split > 768) continue;
    if (!best || k.rb < best->rb || (k.rb == best->rb && k.split > best->split)) best = &k;
  }
  return best;
}

// rows whose degree-1 extension column holds at least one transmitted bit:
// the transmitted mother positions are a prefix of the circular buffer
// (ldpc.py:252-256), so the live rows are a prefix 0..R-1
int live_rows(const QcParams &P) {
  if (P.n >= P.buflen) return P.mb;
  const int last = mother_of(P, P.n - 1);
  const int r = last / P.z - P.kb + 1;
  return r < 4 ? 4 : (r > P.mb ? P.mb : r);
}
}  // namespace lsb

extern "C" int ls_qc_live_rows(const ls_code *code) { return code ? live_rows(code->p) : -1; }

// kernel kind: 0 fp32 min-sum, 1 fp16x2 min-sum, 2 sum-product
static int qc_kind(int variant, int flags) {
  if (variant == LS_SUM_PRODUCT) return (flags & LS_QC_FULL32) ? 3 : 2;
  return (flags & LS_QC_FP16) ? 1 : 0;
}

extern "C" int ls_qc_has_kernel(const ls_code *code, int flags) {
  if (!code) return 0;
  const int R = (flags & LS_QC_PRUNE) ? live_rows(code->p) : code->p.mb;
  const int prec = (flags & LS_QC_SP) ? qc_kind(LS_SUM_PRODUCT, flags) : qc_kind(LS_MIN_SUM, flags);
  if ((flags & LS_QC_EXACT) || ((flags & LS_QC_FULL32) && !(flags & LS_QC_SP))) return find_qcx(code) != nullptr;
  if (!code->std_shifts) return 0;
  for (const QcKernelEntry &k : kQcKernels)
    if (k.bg == code->p.bg && k.z == code->p.z && k.r == R && k.prec == prec) return 1;
  return 0;
}

extern "C" int ls_qc_decode(const ls_code *code, const float *llr, int64_t batch, int num_iter, int variant,
                            double scale, int early_stop, int flags, uint8_t *hard_k, float *llr_out,
                            int32_t *iters_used, const uint8_t *ref_bits, unsigned long long *counts,
                            void *stream) {
  if (!code) return fail(LS_EINVAL, "ls_qc_decode: null code");
  if (variant < 0 || variant > 2) return fail(LS_EINVAL, "unknown BP variant");
  if (num_iter < 1) return fail(LS_EINVAL, "num_iter must be >= 1");
  if (batch <= 0) return LS_OK;
  const QcParams &P = code->p;
  const float alpha = variant == LS_SCALED_MIN_SUM ? (float)scale : 1.0f;
  cudaStream_t s = as_stream(stream);
  if ((flags & LS_QC_EXACT) || ((flags & LS_QC_FULL32) && variant != LS_SUM_PRODUCT)) {
    if (variant == LS_SUM_PRODUCT)
      return fail(LS_EINVAL, "ls_qc_decode: the on-chip exact / fp32 full-graph decoder serves min-sum and "
                             "scaled-min-sum; use ls_bp_decode for sum-product");
    const QcxEntry *k = find_qcx(code);
    if (!k) return fail(LS_EINVAL, "ls_qc_decode: no on-chip exact decoder instance for this code");
    const QcChanParams CP{P.z, P.k, P.n, P.k_full, P.n_full, P.l1, P.buflen};
    const int mother = (flags & LS_QC_MOTHER) ? 1 : 0;
    const QcxFn fn = (flags & LS_QC_EXACT) ? k->fn : k->fn32;
    return fn(CP, llr, batch, num_iter, variant == LS_SCALED_MIN_SUM ? scale : 1.0, early_stop, mother, hard_k,
              mother ? P.n_full : P.k, llr_out, iters_used, ref_bits, counts, s);
  }
  const int prec = qc_kind(variant, flags);
  const int R = (flags & LS_QC_PRUNE) ? live_rows(P) : P.mb;
  const QcChanParams CP{P.z, P.k, P.n, P.k_full, P.n_full, P.l1, P.buflen};
  if (!(flags & LS_QC_GENERIC) && code->std_shifts) {
    for (const QcKernelEntry &k : kQcKernels) {
      if (k.bg == P.bg && k.z == P.z && k.r == R && k.prec == prec)
        return k.fn(CP, llr, batch, num_iter, alpha, early_stop, hard_k, llr_out, iters_used, ref_bits, counts, s);
    }
  }
  if (prec == 3)
    return fail(LS_EINVAL, "ls_qc_decode: no f32 sum-product instance for this (BG, Z, rows); its messages fit "
                           "in shared memory up to Z = 192 with the dead rows pruned");
  if (prec >= 1) {  // fp16x2 / sum-product at any (Z, R): runtime-geometry instance
    const QcRtEntry *k = prec == 1 ? pick_rt(kQcRtKernels, P.bg, P.z, R) : pick_rt(kQcSpRtKernels, P.bg, P.z, R);
    if (!k)
      return fail(LS_EINVAL, prec == 1 ? "ls_qc_decode: no fp16x2 decoder instance for this (BG, Z, rows)"
                                       : "ls_qc_decode: no sum-product fast decoder instance for this (BG, Z, rows); "
                                         "use the exact decoder");
    int32_t col[kMaxNnz];
    for (int e = 0; e < P.nnz; ++e) col[e] = code->entries[3 * e + 1];
    return k->fn(CP, R, P.s, col, llr, batch, num_iter, alpha, early_stop, hard_k, llr_out, iters_used, ref_bits,
                 counts, s);
  }
  QcFastParams FP;
  FP.z = P.z; FP.k = P.k; FP.n = P.n; FP.k_full = P.k_full; FP.n_full = P.n_full; FP.l1 = P.l1;
  FP.buflen = P.buflen;
  FP.nrows = (flags & LS_QC_PRUNE) ? live_rows(P) : P.mb;
  for (int e = 0; e < P.nnz; ++e) {
    const int c = code->entries[3 * e + 1], s = P.s[e];
    FP.thr[e] = P.z - s;
    FP.lo[e] = 4 * (c * P.z + s);
    FP.hi[e] = 4 * (c * P.z + s - P.z);
  }
  if (P.bg == 1)
    return launch_fast<BG1Tables, LS_MIN_SUM>(FP, llr, batch, num_iter, alpha, early_stop, hard_k, llr_out,
                                              iters_used, ref_bits, counts, s);
  return launch_fast<BG2Tables, LS_MIN_SUM>(FP, llr, batch, num_iter, alpha, early_stop, hard_k, llr_out,
                                            iters_used, ref_bits, counts, s);
}
