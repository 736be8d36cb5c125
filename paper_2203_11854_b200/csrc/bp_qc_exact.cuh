// EXACT-mode QC flooding BP decoder, on chip (ldpc.py:86-172 for min-sum and
// scaled-min-sum; ldpc5g_decode ldpc.py:354-365 with derate_match 335-345
// fused in).  Bit-identical to the reference: same f32 posterior rounding,
// f64 messages, numpy add.reduceat summation order, tie rule and per-row
// early stop, with NO dead-row pruning.
//
// Why a compressed check state is exact.  In min-sum every message leaving a
// check is sign * alpha * (min1 or min2) of that check's |v2c| values
// (ldpc.py:144-148, _segment_min2 65-74).  Tracking the multiset minimum
// pair (min1, second smallest with multiplicity) and the first argmin gives
// the reference's result: with a unique minimum the runner-up is the min over
// the other entries, and with a tie it equals min1, which is what the
// reference sends on every edge.  So a check is (alpha*min1, alpha*min2) in
// f64 plus one word with the argmin position and the outgoing sign bits
// (row parity already XORed in); (-alpha)*x == -(alpha*x) exactly, so the
// sign is a bit flip.
//
// Data layout (persistent CTAs; NC codewords per CTA in lockstep, lane
// k * Z + i of every state array = lane i of slot k; NC = 1 at Z = 384):
//   shared  M1 [MB][NC*Z] f64  alpha*min1 of every check
//           W  [MB][NC*Z] u16/u32 outgoing signs (position p at bit deg-1-p)
//                              | argmin, one-hot at bit deg + p for rows of
//                              degree <= 16, else the position << deg
//           T  [KBC][NC*Z] f32 posteriors of the core columns (systematic +
//                              4 core parity; KBC = k_b + 4)
//   global  m2 [MB][NC*Z] f64  alpha*min2 per check, one slice per CTA: read
//                              once per check in the CN phase and once per
//                              argmin edge in the VN phase, L2-resident
//           chn [NC][NB][Z]    channel values -derate(llr) of each slot's
//                              codeword, formed once per codeword (L2)
// Config 2 (BG1, Z = 384): 141,312 + 45,312 + 39,936 = 226,560 B of shared
// memory.  The degree-1 extension columns keep no posterior: their value
// clip(f32(chan + c2v)) is formed inside the check update of their row.
//
// One iteration (flooding, ldpc.py:131-153):
//   CN phase  thread (group g, lane i) walks the rows of its group: old c2v
//             from the compressed state, v2c = f64(total) - c2v_old, new
//             (min1, min2, argmin, signs); the syndrome of the totals it
//             reads is the early-stop test of the PREVIOUS iteration
//             (ldpc.py:155-160), so a converged codeword stops before its
//             next variable update and its posteriors are still in T.
//   VN phase  thread (group g, lane j) walks the core columns of its group:
//             gathers c2v of its column in ascending check order and sums
//             x0 + pairwise(x1..) (numpy reduceat / pairwise_sum), then
//             total = clip(f32(f64(chan) + sum), +-40).
// Rows and core columns are split over NTL thread groups in contiguous,
// degree-balanced ranges; the whole base graph is compile-time, so every
// shift, column and position is an immediate.
#pragma once

#include <math.h>
#include <stdint.h>

#include <type_traits>

#include "bp_fast_qc.cuh"
#include "common.cuh"

namespace lsb {

// M = double: the EXACT decoder (reference arithmetic); M = float: the fp32
// full-graph fast decoder (same schedule and layout with f32 messages, so
// min2 fits in shared memory too).  NC codewords per CTA (slots) run in
// lockstep for Z < 384: every row's code then serves NC * Z lanes, as many
// warps as at Z = 384, and the instruction cache is shared (one codeword of
// Z = 192 per CTA left half the warps per row and stalled on instruction
// fetch, profiles/r02/README.md).
constexpr int qx_default_nc(int z) { return z >= 384 ? 1 : 384 / z; }
#ifndef QX_COL_SHIFT
#define QX_COL_SHIFT -1  // variable-phase column split offset (QxGeo::cfirst)
#endif

template <class G_, int Z_, int NTL_, class M_ = double, int NC_ = qx_default_nc(Z_)>
struct QxGeo {
  using G = G_;
  using M = M_;
  static constexpr bool EXACT = sizeof(M_) == 8;
  static constexpr int Z = Z_, NTL = NTL_, NC = NC_, NZ = NC_ * Z_;
  static constexpr int NT1 = ((NZ + 31) / 32) * 32, NT = NT1 * NTL;
  static constexpr int MB = G::MB, NB = G::NB, KBC = G::KB + 4, NEXT = G::NB - (G::KB + 4);
  static constexpr int MINB = NT >= 768 ? 1 : (NT >= 384 ? 2 : (NT >= 256 ? 4 : 1024 / NT));

  static constexpr int deg(int r) { return G::row_start[r + 1] - G::row_start[r]; }
  static constexpr int cdeg(int c) { return G::col_start[c + 1] - G::col_start[c]; }
  static constexpr int argbits(int d) {
    int b = 0;
    while ((1 << b) < d) ++b;
    return b;
  }
  // argmin as a one-hot field (bit deg + p) when 2 deg <= 32 -- one bit test
  // per edge instead of an extract and compare -- else as an index (<< deg)
  static constexpr bool onehot(int r) { return 2 * deg(r) <= 32; }
  static constexpr int wbits(int r) { return onehot(r) ? 2 * deg(r) : deg(r) + argbits(deg(r)); }
  static constexpr int wbytes(int r) { return wbits(r) <= 16 ? 2 : 4; }
  static constexpr uint32_t argcode(int r, int p) {
    return onehot(r) ? (1u << (deg(r) + p)) : ((uint32_t)p << deg(r));
  }
  // shared: M1 [MB][NZ] M, (fp32: M2 [MB][NZ] M), W, T [KBC][NZ]; lane
  // k * Z + i of a row is lane i of slot k
  static constexpr int M2_OFF = (int)sizeof(M_) * MB * NZ;
  static constexpr int W_OFF = EXACT ? M2_OFF : 2 * M2_OFF;
  static constexpr int woff(int r) {  // byte offset of row r's word array
    int o = W_OFF;
    for (int q = 0; q < r; ++q) {
      if (wbytes(q) == 4) o = (o + 3) & ~3;
      o += wbytes(q) * NZ;
    }
    if (wbytes(r) == 4) o = (o + 3) & ~3;
    return o;
  }
  static constexpr int T_OFF = (woff(MB - 1) + wbytes(MB - 1) * NZ + 15) & ~15;
  static constexpr int SMEM = T_OFF + 4 * KBC * NZ;

  // contiguous degree-balanced ranges: rows [rfirst(g), rfirst(g+1)) and
  // core columns [cfirst(g), cfirst(g+1)) belong to thread group g
  // `shift` moves the group boundaries down the row list: the early-stop
  // kernels' extension rows cost more than their edge count says (syndrome
  // and extension posterior): measured best with the boundary 4 rows later
  // (early stop at 6 dB, Z = 384: 14.18 -> 13.32 ms per 8,192; Z = 192 at
  // 3 dB: 20.15 -> 19.43 ms per 16,384; the fixed-iteration kernels keep 0)
  static constexpr int rfirst(int g, int shift = 0) {
    if (g <= 0) return 0;
    if (g >= NTL) return MB;
    const int tot = G::row_start[MB];
    int r = 0;
    while (r < MB && G::row_start[r] * NTL < tot * g) ++r;
    r += shift;
    return r < MB ? r : MB;
  }
  // variable-node work of core column c in instructions (~13 per edge plus
  // the per-column channel load, sum and store), for balancing the groups
  static constexpr int ccost(int c) { return 13 * cdeg(c) + 16; }
  static constexpr int cfirst(int g) {
    if (g <= 0) return 0;
    if (g >= NTL) return KBC;
    int tot = 0;
    for (int c = 0; c < KBC; ++c) tot += ccost(c);
    int c = 0, acc = 0;
    while (c < KBC && acc * NTL < tot * g) acc += ccost(c++);
    // one column earlier than the cost model says: measured 29.29 -> 29.18 ms
    // (Z = 384, fixed) and 13.30 -> 13.25 ms (early stop); 0, +1, -2, -3 are slower
    c += QX_COL_SHIFT;
    return c > 0 ? c : 0;
  }
  // thread group owning row r / core column c (compile-time only: the
  // tables are host constexpr arrays)
  static constexpr int rowner(int r, int shift = 0) {
    int g = 0;
    while (g + 1 < NTL && r >= rfirst(g + 1, shift)) ++g;
    return g;
  }
  static constexpr int cowner(int c) {
    int g = 0;
    while (g + 1 < NTL && c >= cfirst(g + 1)) ++g;
    return g;
  }
};

// is position p of row r the argmin of the check whose word is w
template <class Geo, int r, int p>
__device__ __forceinline__ bool qx_isarg(uint32_t w) {
  constexpr int D = Geo::deg(r);
  if constexpr (Geo::onehot(r))
    return (w & (1u << (D + p))) != 0u;
  else
    return (w >> D) == (uint32_t)p;
}

// x with its sign bit flipped when `bit31` is 0x80000000 (c2v = (-alpha)*excl)
__device__ __forceinline__ double qx_flip(double x, uint32_t bit31) {
  return __hiloint2double(__double2hiint(x) ^ (int)bit31, __double2loint(x));
}
__device__ __forceinline__ float qx_flip(float x, uint32_t bit31) {
  return __uint_as_float(__float_as_uint(x) ^ bit31);
}
__device__ __forceinline__ double qx_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float qx_add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double qx_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float qx_sub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double qx_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float qx_mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ uint32_t qx_hi(double x) { return (uint32_t)__double2hiint(x); }
__device__ __forceinline__ uint32_t qx_hi(float x) { return __float_as_uint(x); }
__device__ __forceinline__ float qx_to_f32(double x) { return __double2float_rn(x); }
__device__ __forceinline__ float qx_to_f32(float x) { return x; }

// numpy pairwise_sum of N compile-time terms (loops_utils.h.src): fewer
// than 8 terms sequentially from -0.0, else 8 strided accumulators, their
// tree, then the remainder in order
template <int N, class M>
__device__ __forceinline__ M qx_pairwise(const M *x) {
  if constexpr (N < 8) {
    M r = (M)-0.0;
#pragma unroll
    for (int q = 0; q < N; ++q) r = qx_add(r, x[q]);
    return r;
  } else {
    M r[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) r[q] = x[q];
    constexpr int NB8 = N - N % 8;
#pragma unroll
    for (int q = 8; q < NB8; q += 8)
#pragma unroll
      for (int u = 0; u < 8; ++u) r[u] = qx_add(r[u], x[q + u]);
    M res = qx_add(qx_add(qx_add(r[0], r[1]), qx_add(r[2], r[3])), qx_add(qx_add(r[4], r[5]), qx_add(r[6], r[7])));
#pragma unroll
    for (int q = NB8; q < N; ++q) res = qx_add(res, x[q]);
    return res;
  }
}

__device__ __forceinline__ float qx_clip(float x) { return fminf(fmaxf(x, -40.0f), 40.0f); }

// channel value -llr of mother VN v: fused derate_match (rate-matched input)
// or the mother LLRs themselves (bp_decode on the code's pcm)
__device__ __forceinline__ float qx_chan(const QcChanParams &P, const float *__restrict__ row, int v, bool mother) {
  return mother ? -__ldg(row + v) : chan_value(P, row, v);
}

// next codeword of the batch, -1 when it is exhausted
__device__ __forceinline__ long long qx_claim(unsigned long long *next, int64_t batch) {
  const unsigned long long c = atomicAdd(next, 1ULL);
  return (long long)c < batch ? (long long)c : -1;
}

// gather the messages into core column c at lane j of the slot whose lanes
// start at byte k8 / 8 * sizeof(M) (ascending check order): c2v =
// +-(alpha*min1 | alpha*min2) from the compressed state of each check
template <class Geo, int c>
__device__ __forceinline__ void qx_vn_gather(typename Geo::M *x, uint32_t j8, uint32_t k8,
                                             const unsigned char *qx_sm, const typename Geo::M *m2) {
  using G = typename Geo::G;
  using M = typename Geo::M;
  constexpr int Z = Geo::Z, NZ = Geo::NZ, d = Geo::cdeg(c), cs = G::col_start[c], SZ = (int)sizeof(M);
  sfor<0, d>([&](auto tc) {
    constexpr int q = decltype(tc)::value, e = G::col_entry[cs + q], r = G::row[e];
    constexpr int p = e - G::row_start[r], D = Geo::deg(r), s = G::shift[e] % Z;
    using WT = std::conditional_t<Geo::wbytes(r) == 4, uint32_t, uint16_t>;
    uint32_t o8 = j8 - 8u * s;  // 8 * ((j - s) mod Z)
    o8 = min(o8, o8 + 8u * Z);
    if constexpr (Geo::NC > 1) o8 += k8;
    const uint32_t w = *reinterpret_cast<const WT *>(qx_sm + Geo::woff(r) + (o8 >> (sizeof(WT) == 4 ? 1 : 2)));
    const uint32_t oM = SZ == 8 ? o8 : (o8 >> 1);  // byte offset of check (r, lane) in an [MB][NZ] M array
    M mag;
    if (qx_isarg<Geo, r, p>(w)) {
      if constexpr (Geo::EXACT)
        mag = *reinterpret_cast<const M *>(reinterpret_cast<const char *>(m2) + SZ * r * NZ + oM);
      else
        mag = *reinterpret_cast<const M *>(qx_sm + Geo::M2_OFF + SZ * r * NZ + oM);
    } else {
      mag = *reinterpret_cast<const M *>(qx_sm + SZ * r * NZ + oM);
    }
    x[q] = qx_flip(mag, (w << (32 - D + p)) & 0x80000000u);
  });
}

// total = clip(f32(chan + (x0 + pairwise(x1..))), +-40)
template <int d, class M>
__device__ __forceinline__ float qx_vn_total(const M *x, float ch) {
  M sum = x[0];
  if constexpr (d > 1) sum = qx_add(x[0], qx_pairwise<d - 1>(x + 1));
  return qx_clip(qx_to_f32(qx_add((M)ch, sum)));
}

template <class Geo, bool ES, bool OUT>
__global__ void __launch_bounds__(Geo::NT, Geo::MINB)
    k_qc_exact(const QcChanParams P, const float *__restrict__ llr, int64_t batch, int num_iter, double alpha,
               int mother, uint8_t *__restrict__ hard, int hard_len, float *__restrict__ llr_out,
               int32_t *__restrict__ iters_used, const uint8_t *__restrict__ ref,
               unsigned long long *__restrict__ counts, unsigned long long *__restrict__ next,
               typename Geo::M *__restrict__ m2ws, float *__restrict__ extws, float *__restrict__ chws) {
  using G = typename Geo::G;
  using M = typename Geo::M;
  constexpr int Z = Geo::Z, NZ = Geo::NZ, NC = Geo::NC, NT1 = Geo::NT1, NTL = Geo::NTL, MB = Geo::MB;
  constexpr int KBC = Geo::KBC, SLOT_T = NTL * Z;  // threads per slot
#ifndef QX_ES_ROW_SHIFT
#define QX_ES_ROW_SHIFT 4
#endif
#ifndef QX_FX_ROW_SHIFT
#define QX_FX_ROW_SHIFT 0
#endif
  constexpr int RSH = ES ? QX_ES_ROW_SHIFT : QX_FX_ROW_SHIFT;  // row split of the thread groups (rfirst)
  extern __shared__ __align__(16) unsigned char qx_sm[];
  M *M1 = reinterpret_cast<M *>(qx_sm);
  // min2 per check: an L2 slice per CTA for f64 messages, shared memory for f32
  M *m2 = Geo::EXACT ? m2ws + (size_t)blockIdx.x * MB * NZ : reinterpret_cast<M *>(qx_sm + Geo::M2_OFF);
  const M al = (M)alpha;
  float *T = reinterpret_cast<float *>(qx_sm + Geo::T_OFF);
  __shared__ long long cur[NC], nxt[NC];
  __shared__ unsigned errs[NC];
  __shared__ bool rf[NC];  // slot refilled in this refill step
  __shared__ uint32_t flag[2][NC];  // per-slot syndrome flags, double-buffered by CTA iteration
  const int t = threadIdx.x, grp = t / NT1, ln = t - grp * NT1;
  const bool lane = ln < NZ;
  const int k = NC == 1 || !lane ? 0 : ln / Z;  // slot
  const int i = ln - k * Z;         // lane within the slot's codeword
  const int ts = grp * Z + i;       // thread index within the slot
  float *ext = OUT ? extws + (size_t)blockIdx.x * Geo::NEXT * NZ : nullptr;
  // channel values -derate(llr) of the slot's codeword, formed once per
  // codeword (fillers, punctured positions, repetitions) and re-read from L2
  float *chn = chws + ((size_t)blockIdx.x * NC + k) * Geo::NB * Z;
  const bool moth = mother != 0;
  const int row_len = moth ? P.n_full : P.n;
  const uint32_t k4 = 4u * (uint32_t)(k * Z), k8 = 2u * k4;  // byte offsets of the slot's lanes
  // per-thread bases, so that every row / column offset is an immediate
  M *const M1l = M1 + ln;
  M *const m2l = m2 + ln;
  const float *const chj = chn + i;
  float *const Tkj = T + k * Z + i;

  if (t < NC) flag[0][t] = flag[1][t] = 0u;
  long long cw = -1;
  int it = 0, used = 0;
  bool need = lane;     // the slot wants a new codeword
  bool refill = true;  // CTA-uniform: some slot finished in the last iteration
  for (int g = 0;; ++g) {
    if (refill) {
      // ------------------------------------------------ refill finished slots
      // (claimed one codeword ahead: the next one's LLR row is prefetched
      // into L2 while this one decodes, so the refill's loads hit L2)
      if (lane && ts == 0) {
        if (need) {
          const long long c = g == 0 ? qx_claim(next, batch) : nxt[k];
          cur[k] = c;
          nxt[k] = c >= 0 ? qx_claim(next, batch) : -1;
          errs[k] = 0u;
        }
        rf[k] = need;
      }
      __syncthreads();
      if (NC == 1) it = 0;  // one slot: keep the iteration state CTA-uniform
      if (need) {
        need = false;
        cw = cur[k];
        it = 0;
        const long long nx = nxt[k];
        if (nx >= 0) {
          const char *nrow = reinterpret_cast<const char *>(llr + nx * (int64_t)row_len);
          for (int b = 128 * ts; b < 4 * row_len; b += 128 * SLOT_T) asm volatile("prefetch.global.L2 [%0];" ::"l"(nrow + b));
          if (ref && 128 * ts < P.k)  // and its reference bits (one line per thread)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(ref + nx * (int64_t)P.k + 128 * ts));
        }
        if (cw >= 0) {
          // zero check state: the first iteration's old messages are +0
          if constexpr (!(ES && NC == 1)) sfor<0, MB>([&](auto rc) {
            constexpr int r = decltype(rc)::value;
            if (grp != Geo::rowner(r, RSH)) return;
            using WT = std::conditional_t<Geo::wbytes(r) == 4, uint32_t, uint16_t>;
            M1l[r * NZ] = (M)0;
            m2l[r * NZ] = (M)0;
            reinterpret_cast<WT *>(qx_sm + Geo::woff(r))[ln] = (WT)0;
          });
          if constexpr (NC == 1) {
            const float *row = llr + cw * (int64_t)row_len;
#pragma unroll 4
            for (int v = ts; v < Geo::NB * Z; v += SLOT_T) {
              const float ch = qx_chan(P, row, v, moth);
              chn[v] = ch;
              const int c = v / Z;
              if (c < KBC) T[c * NZ + (v - c * Z)] = ch;
            }
          }
        }
      }
      if constexpr (NC > 1) {
        // the channel values of every refilled slot, by all threads of the
        // CTA (the other slots wait at the next barrier anyway): the load is
        // latency-bound, so more threads per codeword shorten it
        for (int kk = 0; kk < NC; ++kk) {
          const long long ck = rf[kk] ? cur[kk] : -1;  // CTA-uniform
          if (ck < 0) continue;
          const float *row = llr + ck * (int64_t)row_len;
          float *chk = chws + ((size_t)blockIdx.x * NC + kk) * Geo::NB * Z;
#pragma unroll 4
          for (int v = t; v < Geo::NB * Z; v += Geo::NT) {
            const float ch = qx_chan(P, row, v, moth);
            chk[v] = ch;
            const int c = v / Z;
            if (c < KBC) T[c * NZ + kk * Z + (v - c * Z)] = ch;
          }
        }
      }
      if (!__syncthreads_or(lane && cw >= 0)) return;
    }
    // (one slot: the CTA returned above unless its codeword is live)
    const bool act = NC == 1 ? lane : lane && cw >= 0;
    const bool first = it == 0;
    uint32_t bad = 0;
    // ------------------------------------------------ check-node phase
    if (act) {
      uint32_t i4 = 4u * (uint32_t)i;
      // opaque per iteration: keeps the ~600 per-edge lane offsets from
      // being hoisted out of the iteration loop (and spilled)
      asm volatile("" : "+r"(i4));
      const char *Tk = reinterpret_cast<const char *>(T) + k4;
      sfor<0, MB>([&](auto rc) {
        constexpr int r = decltype(rc)::value;
        if (grp != Geo::rowner(r, RSH)) return;  // warp-uniform
        constexpr int e0 = G::row_start[r], D = Geo::deg(r);
        using WT = std::conditional_t<Geo::wbytes(r) == 4, uint32_t, uint16_t>;
        WT *W = reinterpret_cast<WT *>(qx_sm + Geo::woff(r));
        // old messages are +0 in the first iteration: a refilled slot's state
        // is zeroed (no branch in the hot loop, slots stay in step), except
        // for one-slot early-stop kernels, which skip the loads (a different
        // register allocation wins there)
        M m1o = 0, m2o = 0;
        uint32_t wo = 0u;
        if (!(ES && NC == 1) || !first) {
          m1o = M1l[r * NZ];
          m2o = m2l[r * NZ];
          wo = (uint32_t)W[ln];
        }
        M mn1 = (M)INFINITY, mn2 = (M)INFINITY;
        uint32_t arg = 0, sg = 0, syn = 0;
        sfor<0, D>([&](auto pc) {
          constexpr int p = decltype(pc)::value, e = e0 + p, c = G::col[e], s = G::shift[e] % Z;
          // old message on this edge: +-(alpha*min1 | alpha*min2), sign
          // bit of position p at bit D-1-p of the word
          const M mag = qx_isarg<Geo, r, p>(wo) ? m2o : m1o;
          const M cold = qx_flip(mag, (wo << (32 - D + p)) & 0x80000000u);
          uint32_t o = i4 + 4u * s;  // byte offset of lane (i + s) mod Z
          o = min(o, o - 4u * Z);
          float tv;
          if constexpr (c < KBC) {
            tv = *reinterpret_cast<const float *>(Tk + 4 * c * NZ + o);
          } else {
            // degree-1 extension VN: its posterior is chan + its only message
            const int v = c * Z + (int)(o >> 2);
            const float ch = chn[v];
            tv = first ? ch : qx_clip(qx_to_f32(qx_add((M)ch, cold)));
            if (OUT && ES) ext[(c - KBC) * NZ + k * Z + (int)(o >> 2)] = tv;
          }
          if (ES) syn ^= __float_as_uint(tv);
          const M x = qx_sub((M)tv, cold);
          if constexpr (Geo::EXACT) {
            const double a = fabs(x);
            const bool lt1 = a < mn1, lt2 = a < mn2;
            const double t2 = lt2 ? a : mn2;
            mn2 = lt1 ? mn1 : t2;
            mn1 = lt1 ? a : mn1;
            arg = lt1 ? Geo::argcode(r, p) : arg;
          } else {  // one FMNMX per update in f32
            const float a = fabsf(x);
            arg = a < mn1 ? Geo::argcode(r, p) : arg;
            mn2 = fminf(mn2, fmaxf(mn1, a));
            mn1 = fminf(mn1, a);
          }
          sg = __funnelshift_l(qx_hi(x), sg, 1);  // signbit(x) in at bit 0
        });
        bad |= syn >> 31;
        const uint32_t osg = (__popc(sg) & 1) ? sg ^ ((1u << D) - 1u) : sg;
        M1l[r * NZ] = qx_mul(al, mn1);
        m2l[r * NZ] = qx_mul(al, mn2);
        W[ln] = (WT)(osg | arg);
      });
    }
    // the slot's codeword passed the syndrome of the posteriors of its
    // iteration `it` (ldpc.py:155-160): it stops before the variable update
    bool conv = false;
    if constexpr (ES && NC == 1) {
      conv = !__syncthreads_or(bad) && !first;
    } else {
      if (ES && bad) flag[g & 1][k] = 1u;
      __syncthreads();
      if (ES) {
        conv = act && !first && flag[g & 1][k] == 0u;
        if (t < NC) flag[(g + 1) & 1][t] = 0u;
      }
    }
    // ------------------------------------------------ variable-node phase
    if (act && !conv) {
      const int j = i;
      uint32_t j8 = 8u * (uint32_t)j;
      asm volatile("" : "+r"(j8));
      sfor<0, KBC>([&](auto cc) {
        constexpr int c = decltype(cc)::value;
        if (grp != Geo::cowner(c)) return;  // warp-uniform
        const float ch = chj[c * Z];
        M x[Geo::cdeg(c)];
        qx_vn_gather<Geo, c>(x, j8, k8, qx_sm, m2);
        Tkj[c * NZ] = qx_vn_total<Geo::cdeg(c)>(x, ch);
      });
    }
    bool fin = false;
    if (NC == 1 || act) {
      if (conv) {
        used = it;
        fin = true;
      } else if (++it == num_iter) {
        used = num_iter;
        fin = true;
      }
    }
    refill = __syncthreads_or(fin);
    if (!refill) continue;

    // ------------------------------------------------ outputs of finished slots
    if (OUT) {
      // extension posteriors after the last variable update: chan + c2v
      if (fin && used == num_iter) {
        sfor<4, MB>([&](auto rc) {
          constexpr int r = decltype(rc)::value;
          if (grp != Geo::rowner(r, RSH)) return;
          constexpr int D = Geo::deg(r), e = G::row_start[r + 1] - 1, c = G::col[e], s = G::shift[e] % Z;
          if constexpr (c >= KBC) {
            using WT = std::conditional_t<Geo::wbytes(r) == 4, uint32_t, uint16_t>;
            const WT *W = reinterpret_cast<const WT *>(qx_sm + Geo::woff(r));
            const uint32_t w = W[ln];
            const M mag = qx_isarg<Geo, r, D - 1>(w) ? m2[r * NZ + ln] : M1[r * NZ + ln];
            const M cv = qx_flip(mag, (w << 31) & 0x80000000u);  // position D-1: bit 0
            int jj = i + s;
            jj = jj >= Z ? jj - Z : jj;
            const float ch = chn[c * Z + jj];
            ext[(c - KBC) * NZ + k * Z + jj] = qx_clip(qx_to_f32(qx_add((M)ch, cv)));
          }
        });
      }
      __syncthreads();
    }
    if (fin) {
      if (iters_used && ts == 0) iters_used[cw] = used;
      auto post = [&](int v) -> float {  // posterior of mother VN v of the slot's codeword
        const int c = v / Z, jj = v - c * Z;
        return c < KBC ? T[c * NZ + k * Z + jj] : (OUT ? ext[(c - KBC) * NZ + k * Z + jj] : 0.0f);
      };
      if (OUT && llr_out) {
        float *o = llr_out + cw * (int64_t)P.n_full;
        for (int v = ts; v < P.n_full; v += SLOT_T) o[v] = -post(v);
      }
      unsigned err = 0;
      if (!hard && ref && (P.k & 3) == 0) {
        // error count only: the reference bits four at a time
        const uint32_t *rw = reinterpret_cast<const uint32_t *>(ref + cw * (int64_t)P.k);
        for (int w = ts; w < (P.k >> 2); w += SLOT_T) {
          const uint32_t r4 = rw[w];
#pragma unroll
          for (int q = 0; q < 4; ++q) err += (uint32_t)((-post(4 * w + q)) > 0.0f) != ((r4 >> (8 * q)) & 0xffu);
        }
      } else if (hard || ref) {
        for (int v = ts; v < hard_len; v += SLOT_T) {
          const uint8_t h = (-post(v)) > 0.0f;
          if (hard) hard[cw * (int64_t)hard_len + v] = h;
          if (ref && v < P.k) err += (h != ref[cw * (int64_t)P.k + v]);
        }
      }
      if (ref && counts && err) atomicAdd(&errs[k], err);
      need = true;
    }
    if (ref && counts) {
      __syncthreads();
      if (fin && ts == 0 && errs[k]) {
        atomicAdd(&counts[0], (unsigned long long)errs[k]);
        atomicAdd(&counts[1], 1ULL);
      }
    }
  }
}

// one decoder instance: persistent grid of NC-slot CTAs; the exact (f64)
// decoder keeps an L2 slice of min2 per CTA, the fp32 one keeps everything
// but the channel in shared memory
template <class G, int Z, int NTL, class M = double>
int launch_qc_exact(const QcChanParams &P, const float *llr, int64_t B, int num_iter, double alpha, int early_stop,
                    int mother, uint8_t *hard, int hard_len, float *llr_out, int32_t *iters_used, const uint8_t *ref,
                    unsigned long long *counts, cudaStream_t s) {
  using Geo = QxGeo<G, Z, NTL, M>;
  static_assert(Geo::SMEM <= 227 * 1024, "decoder state does not fit in shared memory");
  const bool out = llr_out != nullptr || hard_len > Geo::KBC * Z;
  auto kern = early_stop ? (out ? k_qc_exact<Geo, true, true> : k_qc_exact<Geo, true, false>)
                         : (out ? k_qc_exact<Geo, false, true> : k_qc_exact<Geo, false, false>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Geo::SMEM);
  if (e != cudaSuccess) return cuda_status(e, "ls_qc_decode(exact smem attr)");
  if (num_iter < 1) return fail(LS_EINVAL, "num_iter must be >= 1");  // the slot loop needs one iteration
  if (B <= 0) return LS_OK;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Geo::NT, Geo::SMEM);
  // enough CTAs for every slot to start with a codeword when the batch is small
  const int64_t grid = std::min<int64_t>((int64_t)sms * std::max(1, per_sm), (B + Geo::NC - 1) / Geo::NC);
  const size_t m2_bytes = Geo::EXACT ? sizeof(M) * (size_t)grid * Geo::MB * Geo::NZ : 0;
  const size_t ext_bytes = out ? sizeof(float) * (size_t)grid * Geo::NEXT * Geo::NZ : 0;
  const size_t ch_bytes = sizeof(float) * (size_t)grid * Geo::NB * Geo::NZ;
  char *ws = nullptr;
  retain_pool_memory();
  e = cudaMallocAsync((void **)&ws, 256 + m2_bytes + ext_bytes + ch_bytes, s);
  if (e != cudaSuccess) return cuda_status(e, "ls_qc_decode(exact workspace)");
  unsigned long long *next = reinterpret_cast<unsigned long long *>(ws);
  cudaMemsetAsync(next, 0, sizeof(unsigned long long), s);
  M *m2 = reinterpret_cast<M *>(ws + 256);
  float *ext = out ? reinterpret_cast<float *>(ws + 256 + m2_bytes) : nullptr;
  float *chn = reinterpret_cast<float *>(ws + 256 + m2_bytes + ext_bytes);
  kern<<<(unsigned)grid, Geo::NT, Geo::SMEM, s>>>(P, llr, B, num_iter, alpha, mother, hard, hard_len, llr_out,
                                                   iters_used, ref, counts, next, m2, ext, chn);
  e = cudaGetLastError();
  cudaFreeAsync(ws, s);
  return e == cudaSuccess ? LS_OK : cuda_status(e, "ls_qc_decode(exact)");
}

}  // namespace lsb
