// FAST-mode QC decoder, packed fp16x2 variant (F4): every 32-bit lane word
// carries the same message of TWO codewords (A in the low half, B in the
// high half), so one instruction advances both.  Structure, schedule and
// compile-time specialisation are those of k_qc_fast2 (bp_fast_qc.cuh);
// the differences are the packed state and arithmetic:
//   posterior   half2 {A, B} per VN in shared memory
//   CN state    M1, M2 = half2 {min_A, min_B} (alpha-scaled), IX = half2
//               {argmin_A, argmin_B} (small integers are exact in fp16), sign
//               bits A: bits 0..15, B: 16..31 of one word (edges 0..15) and of
//               a second word (edges 16..31) for rows of degree above 16
//   per edge    mag   = select(M1, M2, IX == {p,p})        (HSET2 + LOP3)
//               cold  = mag | signs moved to bits 15/31     (SHF + LOP3)
//               x     = t - cold                            (HADD2)
//               min1/min2/argmin update                     (HMNMX2, HSET2, LOP3)
// Precision: fp16 (11-bit significand) messages and posteriors, as in
// production 5G decoders; statistically equivalent to the reference and
// checked like the fp32 kernel (tests/test_gpu_parity.py).
#pragma once

#include <cuda_fp16.h>

#include <algorithm>

#include "bp_fast_qc.cuh"

namespace lsb {

__device__ __forceinline__ uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t *>(&h); }
__device__ __forceinline__ __half2 u2h(uint32_t u) { return *reinterpret_cast<__half2 *>(&u); }

__host__ __device__ constexpr int ilog2c(int p) { return p > 1 ? 1 + ilog2c(p >> 1) : 0; }

// half2 {p, p} bit pattern of a small non-negative integer, at compile time
template <int P>
__device__ __forceinline__ constexpr uint32_t h2_int() {
  static_assert(P >= 0 && P < 2048, "integer not exact in fp16");
  if constexpr (P == 0) {
    return 0u;
  } else {
    constexpr int e = ilog2c(P);
    constexpr uint32_t h = ((uint32_t)(e + 15) << 10) | (((uint32_t)P - (1u << e)) << (10 - e));
    return h | (h << 16);
  }
}

template <class G, int Z, int R, int SPLIT>
struct QcShapeH2 {
  static constexpr int NT1 = ((Z + 31) / 32) * 32;
  static constexpr int NT = NT1 * SPLIT;
  static constexpr int NCOL = G::KB + (R > 4 ? R : 4);
  static constexpr int NV = NCOL * Z;
  static constexpr int NR = (R + SPLIT - 1) / SPLIT;
  static constexpr size_t ARR = 4 * (size_t)NV;  // one half2 per VN
  static constexpr bool CHN_SMEM = (SPLIT + 1) * ARR <= 225 * 1024;
  static constexpr size_t SMEM = (SPLIT + (CHN_SMEM ? 1 : 0)) * ARR;
  static constexpr int MINB = NT >= 384 ? 1 : (384 / NT);
};

// Geometry policies.  The phase functions and kernels below are written once
// against a policy `Geo`:
//   H2GeoCT<G, Z, R, SPLIT>  everything compile-time (the specialised
//                            instances of qc_instances.h): shifts, column
//                            bases and loop bounds are immediates;
//   H2GeoRT<G, RB, SPLIT>    base-graph structure and a row bound RB
//                            compile-time; Z, the processed rows R <= RB and
//                            the per-edge shift / column offsets are runtime
//                            values held in the kernel's parameter space, so
//                            they are constant-bank operands (one extra IADD
//                            per edge visit against the immediate form).
template <class G_, int Z, int R, int SPLIT_>
struct H2GeoCT {
  using G = G_;
  using S = QcShapeH2<G_, Z, R, SPLIT_>;
  static constexpr int SPLIT = SPLIT_, RB = R, NR = S::NR, NT_MAX = S::NT, MINB = S::MINB;
  __device__ __forceinline__ static constexpr int nt1() { return S::NT1; }
  __device__ __forceinline__ static constexpr int nt() { return S::NT; }
  __device__ __forceinline__ static constexpr int nv() { return S::NV; }
  __device__ __forceinline__ static constexpr bool chn_smem() { return S::CHN_SMEM; }
  __device__ __forceinline__ static constexpr int z() { return Z; }
  // every thread of a slot serves a lane (Z a multiple of 32)
  __device__ __forceinline__ static constexpr bool full_lanes() { return S::NT1 == Z; }
  template <int r>
  __device__ __forceinline__ static constexpr bool live() { return true; }
  template <int e>
  __device__ __forceinline__ static unsigned off(unsigned i4) { return vn_off<G_, Z, e>(i4); }
  template <int e>
  __device__ __forceinline__ static unsigned coff(unsigned i4) { return vn_off<G_, Z, e>(i4); }
};

// Wrap-free layout of the fixed-iteration D1 kernel (k_qc_fast_h2w): the
// posteriors of the NCA = k_b + 4 accumulated columns are stored twice per
// column (2Z words, word Z + j = word j), and so are the channel words of the
// degree-1 extension columns, so the check-node read of VN (c, (i + s) mod Z)
// is the word c*2Z + i + s: the lane offset plus an immediate, no wrap.
//   T   [NCA][2Z]             posteriors; the accumulators of slots 0 and 1
//   A   [SPLIT-2][NCA][Z]     accumulators of slots 2..SPLIT-1
//   C   [NCA][Z] ++ [NCD][2Z] channel words (extension columns doubled)
template <class G_, int Z, int R, int SPLIT_>
struct H2GeoCTW : H2GeoCT<G_, Z, R, SPLIT_> {
  using G = G_;
  static constexpr int NCA = G_::KB + 4, NCD = R > 4 ? R - 4 : 0;
  static constexpr int T_W = NCA * 2 * Z, A_W = NCA * Z;
  static constexpr int C_OFF = T_W + (SPLIT_ > 2 ? SPLIT_ - 2 : 0) * A_W;  // channel region, in words
  // first word of slot q's accumulator for column c (see h2w_vn)
  __host__ __device__ static constexpr int acc_word(int q, int c) {
    return q == 0 ? c * 2 * Z : (q == 1 ? c * 2 * Z + Z : T_W + (q - 2) * A_W + c * Z);
  }
  static constexpr int C_W = NCA * Z + NCD * 2 * Z;
  static constexpr size_t SMEM = 4 * (size_t)(C_OFF + C_W);
  static constexpr bool FITS = SMEM <= 225 * 1024;
  // small lifting sizes with few rows per thread: aim for 1,024 resident
  // threads per SM (the compact layout leaves the shared memory for it; the
  // register cap becomes 64, enough for <= 6 rows of check state)
  static constexpr int MINB = (H2GeoCT<G_, Z, R, SPLIT_>::NT_MAX < 768 && H2GeoCT<G_, Z, R, SPLIT_>::NR <= 6)
                                  ? 1024 / H2GeoCT<G_, Z, R, SPLIT_>::NT_MAX
                                  : H2GeoCT<G_, Z, R, SPLIT_>::MINB;
  template <int e>
  __device__ __forceinline__ static unsigned off(unsigned i4) {
    constexpr unsigned c = (unsigned)G_::col[e], s = (unsigned)(G_::shift[e] % Z);
    static_assert(G_::col[e] < NCA, "wrap-free read of an extension column");
    return 4u * (c * 2u * Z + s) + i4;
  }
  template <int e>
  __device__ __forceinline__ static unsigned coff(unsigned i4) {
    constexpr unsigned c = (unsigned)G_::col[e], s = (unsigned)(G_::shift[e] % Z);
    static_assert(G_::col[e] >= NCA, "doubled channel words exist for extension columns only");
    return 4u * ((unsigned)NCA * Z + (c - NCA) * 2u * Z + s) + i4;
  }
};

template <class G_, int RB_, int SPLIT_>
struct H2GeoRT {
  using G = G_;
  static constexpr int SPLIT = SPLIT_, RB = RB_, NR = (RB_ + SPLIT_ - 1) / SPLIT_;
  static constexpr int NE = G_::row_start[RB_];  // edges of rows < RB
  static constexpr int NT_MAX = 768, MINB = 1;   // Z <= 384 / SPLIT * 2 (launcher checks)
  int Z, NT1, NT, NV, R, CHN;
  unsigned Z4;
  uint32_t s4[NE];  // 4 * (shift mod Z)
  uint32_t cb[NE];  // 4 * Z * column
  __device__ __forceinline__ int nt1() const { return NT1; }
  __device__ __forceinline__ int nt() const { return NT; }
  __device__ __forceinline__ int nv() const { return NV; }
  __device__ __forceinline__ bool chn_smem() const { return CHN != 0; }
  __device__ __forceinline__ int z() const { return Z; }
  __device__ __forceinline__ static constexpr bool full_lanes() { return false; }
  template <int r>
  __device__ __forceinline__ bool live() const { return r < R; }
  template <int e>
  __device__ __forceinline__ unsigned off(unsigned i4) const {
    const unsigned u = i4 + s4[e];
    return cb[e] + min(u, u - Z4);
  }
  template <int e>
  __device__ __forceinline__ unsigned coff(unsigned i4) const {
    return off<e>(i4);
  }
};

// per-codeword outputs of half `hb` (0 = A, 1 = B) from the current posteriors
template <int NT_MAX>
__device__ __forceinline__ void h2_emit(const QcChanParams &P, const uint32_t *tot, int nv, int NT, int64_t cw,
                                        const float *row, int hb, int used, uint8_t *hard_k, float *llr_out,
                                        int32_t *iters_used, const uint8_t *ref, unsigned long long *counts,
                                        unsigned *red) {
  const int t = threadIdx.x;
  if (iters_used && t == 0) iters_used[cw] = used;
  if (llr_out) {
    float *o = llr_out + cw * (int64_t)P.n_full;
    for (int v = t; v < P.n_full; v += NT) {
      float val;
      if (v < nv) {
        const uint32_t w = tot[v];
        val = -__half2float(__ushort_as_half((unsigned short)(hb ? (w >> 16) : (w & 0xFFFFu))));
      } else {
        val = -chan_value(P, row, v);
      }
      o[v] = val;
    }
  }
  unsigned err = 0;
  for (int v = t; v < P.k; v += NT) {
    const uint32_t w = tot[v];
    const unsigned short hv = (unsigned short)(hb ? (w >> 16) : (w & 0xFFFFu));
    const uint8_t hd = (-__half2float(__ushort_as_half(hv))) > 0.0f;
    if (hard_k) hard_k[cw * (int64_t)P.k + v] = hd;
    if (ref) err += (hd != ref[cw * (int64_t)P.k + v]);
  }
  if (ref && counts) {
#pragma unroll
    for (int o = 16; o; o >>= 1) err += __shfl_xor_sync(0xffffffffu, err, o);
    if ((t & 31) == 0) red[t >> 5] = err;
    __syncthreads();
    if (t == 0) {
      unsigned long long tt = 0;
      for (int w = 0; w < (NT + 31) / 32; ++w) tt += red[w];
      if (tt) {
        atomicAdd(&counts[0], tt);
        atomicAdd(&counts[1], 1ULL);
      }
    }
    __syncthreads();
  }
}

// per-thread compressed check state of the thread's NR rows (registers once
// the phase functions are inlined with compile-time row indices)
// base entry e sits in a degree-1 column (an extension parity bit): its
// variable hears from no other check, so posterior - own message = channel
template <class G, int E>
__host__ __device__ constexpr bool col_deg1() {
  return G::col_start[G::col[E] + 1] - G::col_start[G::col[E]] == 1;
}

// Sign bits of a row's edges: edge p < 16 in SG (codeword A at bit p, B at
// bit 16 + p), edges 16..31 the same way in SG2, so every edge's sign moves
// to the fp16 sign positions with one shift and a mask.
template <int P>
__device__ __forceinline__ uint32_t old_sign(uint32_t osg, uint32_t osg2) {
  static_assert(P < 32, "row degree above 32");
  constexpr int Q = P & 15;
  return ((P < 16 ? osg : osg2) << (15 - Q)) & 0x80008000u;
}
template <int P>
__device__ __forceinline__ void acc_sign(uint32_t &sg, uint32_t &sg2, uint32_t xw) {
  constexpr int Q = P & 15;
  uint32_t &t = P < 16 ? sg : sg2;
  if constexpr (Q == 15)
    t |= xw & 0x80008000u;
  else
    t |= __umulhi(xw, 1u << (17 + Q)) & (0x10001u << Q);  // xw >> (15 - Q)
}

template <int NR>
struct H2State {
  uint32_t M1[NR], M2[NR], IX[NR], SG[NR], SG2[NR];
};

// Check-node phase of one iteration for the calling thread's rows; returns
// the OR of the row syndromes (bit 15: codeword A, bit 31: codeword B), or 0
// when SYN is off (fixed-iteration decoding needs no syndrome).
// D1 (no posterior output requested): an edge into a degree-1
// extension-parity variable takes its variable-to-check message straight
// from the cached channel word -- the min-sum value posterior - own message
// without the fp16 round trip -- and those variables' posteriors are never
// formed (h2_vn skips them); with SYN their syndrome sign is channel + own
// message, the same fp16 sum the variable update would have stored.
template <class Geo, bool SYN = true, bool D1 = false>
__device__ __forceinline__ uint32_t h2_cn(H2State<Geo::NR> &st, const char *base, int h, bool lane, __half2 al2,
                                         bool scaled, const Geo &geo, const char *cbase = nullptr) {
  using G = typename Geo::G;
  constexpr int SPLIT = Geo::SPLIT, NR = Geo::NR;
  uint32_t synx = 0;
  if (!lane) return 0;
  sfor<0, SPLIT>([&](auto hc) {
    constexpr int H = decltype(hc)::value;
    if (h != H) return;
    const unsigned i4 = 4u * tid_volatile() - 4u * H * geo.nt1();
    sfor<0, NR>([&](auto jc) {
      constexpr int j = decltype(jc)::value;
      constexpr int r = j * SPLIT + H;
      if constexpr (r < Geo::RB) {
        if (!geo.template live<r>()) return;
        constexpr int e0 = G::row_start[r], e1 = G::row_start[r + 1], d = e1 - e0;
        constexpr bool packed = d <= 16;
        // ALU-pipe relief: the min1/min2 select is an fp16 FMA on a 1.0/0.0
        // compare result (FMA pipe)
        const __half2 o1 = u2h(st.M1[j]), od = u2h(st.M2[j]), oix = u2h(st.IX[j]);
        const uint32_t osg = st.SG[j], osg2 = st.SG2[j];
        uint32_t n1 = 0x7C007C00u, n2 = 0x7C007C00u, sg = 0u, sg2 = 0u;
        __half2 wv = u2h(0u);
        [[maybe_unused]] uint32_t hs = 0u;
        sfor<e0, e1>([&](auto ec) {
          constexpr int e = decltype(ec)::value;
          constexpr int p = e - e0;
          __half2 x;
          if constexpr (D1 && col_deg1<G, e>()) {
            const uint32_t cw = *reinterpret_cast<const uint32_t *>(cbase + geo.template coff<e>(i4));
            x = u2h(cw);
            if constexpr (SYN) {  // the unformed posterior's sign: channel + own message
              const uint32_t mag = h2u(__hfma2(__heq2(oix, u2h(h2_int<p>())), od, o1));
              hs ^= h2u(__hadd2(u2h(cw), u2h(mag ^ old_sign<p>(osg, osg2))));
            }
          } else {
            const uint32_t tw = *reinterpret_cast<const uint32_t *>(base + geo.template off<e>(i4));
            if constexpr (SYN) hs ^= tw;
            const __half2 pp = u2h(h2_int<p>());
            const uint32_t mag = h2u(__hfma2(__heq2(oix, pp), od, o1));
            x = __hsub2(u2h(tw), u2h(mag ^ old_sign<p>(osg, osg2)));
          }
          const uint32_t xw = h2u(x);
          const __half2 a = __habs2(x);
          // argmin on the FMA pipe: w = argmin - p, kept as w' = u (w - 1)
          // with u = (a >= min1) in {0, 1} (HSET2.BF + HFMA2), so a new
          // minimum (u = 0) resets it to 0; first minimum wins.  The first
          // two edges start from min1 = min2 = +inf, which the compiler
          // cannot fold through HMNMX2, so they are written out.
          if constexpr (p == 0) {
            n1 = h2u(a);  // n2 stays +inf, argmin 0
          } else if constexpr (p == 1) {
            const __half2 u = __hge2(a, u2h(n1));
            wv = __hneg2(u);
            n2 = h2u(__hmax2(u2h(n1), a));
            n1 = h2u(__hmin2(u2h(n1), a));
          } else {
            const __half2 u = __hge2(a, u2h(n1));
            wv = __hfma2(u, wv, __hneg2(u));
            n2 = h2u(__hmin2(u2h(n2), __hmax2(u2h(n1), a)));
            n1 = h2u(__hmin2(u2h(n1), a));
          }
          acc_sign<p>(sg, sg2, xw);
        });
        // The outgoing sign of edge p is (its v2c sign) XOR (row parity): the
        // raw v2c signs are stored and the parity rides in the sign bits of
        // M1 and M2 - M1 (both halves), so reconstruction is
        // fma(eq, D, M1) ^ raw sign -- one parity computation per row, no
        // per-row flip of the sign words.
        uint32_t pa, pb;
        if constexpr (packed) {
          pa = __popc(sg & 0xFFFFu);
          pb = __popc(sg >> 16);
        } else {
          pa = __popc(sg & 0xFFFFu) + __popc(sg2 & 0xFFFFu);
          pb = __popc(sg >> 16) + __popc(sg2 >> 16);
        }
        const uint32_t par = ((pa << 15) & 0x8000u) | (pb << 31);
        st.SG[j] = sg;
        if constexpr (!packed) st.SG2[j] = sg2;
        if (scaled) {
          n1 = h2u(__hmul2(u2h(n1), al2));
          n2 = h2u(__hmul2(u2h(n2), al2));
        }
        // state keeps min1 and the fp16 difference min2 - min1; the argmin
        // edge is reconstructed as min1 + diff (within 1 ulp of min2)
        st.M1[j] = n1 | par;
        st.M2[j] = h2u(__hsub2(u2h(n2), u2h(n1))) | par;
        st.IX[j] = d > 1 ? h2u(__hadd2(wv, u2h(h2_int<d - 1>()))) : 0u;
        if constexpr (SYN) synx |= hs;
      }
    });
  });
  return synx;
}

// Variable-node phase: posteriors = clip(chan + sum of the new messages).
// `chan_word(v)` supplies the channel half2 of VN v when it is not cached.
template <class Geo, bool D1 = false, class ChanFn>
__device__ __forceinline__ void h2_vn(const H2State<Geo::NR> &st, uint32_t *tot, const uint32_t *chn, char *base,
                                      int h, bool lane, int t, ChanFn chan_word, const Geo &geo) {
  using G = typename Geo::G;
  constexpr int SPLIT = Geo::SPLIT, NR = Geo::NR;
  const int NVA = geo.nv(), NT = geo.nt();
  // with D1 only the columns left of the degree-1 extension parities are
  // reset / accumulated / combined (array strides stay NVA)
  const int NV = D1 ? (G::KB + 4) * geo.z() : NVA;
  if (geo.chn_smem() && NV % 4 == 0 && NVA % 4 == 0) {
    // 128-bit shared accesses: 4 posteriors (8 messages) per instruction
    uint4 *t4 = reinterpret_cast<uint4 *>(tot);
    const uint4 *c4 = reinterpret_cast<const uint4 *>(chn);
    for (int v = t; v < NV / 4; v += NT) {
      t4[v] = c4[v];
#pragma unroll
      for (int q = 1; q < SPLIT; ++q) t4[q * (NVA / 4) + v] = make_uint4(0u, 0u, 0u, 0u);
    }
  } else {
    for (int v = t; v < NV; v += NT) {
      tot[v] = geo.chn_smem() ? chn[v] : chan_word(v);
#pragma unroll
      for (int q = 1; q < SPLIT; ++q) tot[q * NVA + v] = 0u;
    }
  }
  __syncthreads();
  // slot H accumulates its rows into its own array, one row per barrier step
  // (consecutive rows of a slot may share variables); every slot passes the
  // same NR barriers, so the slot branch is taken once per phase
  sfor<0, SPLIT>([&](auto hc) {
    constexpr int H = decltype(hc)::value;
    if (h != H) return;
    const unsigned i4 = 4u * tid_volatile() - 4u * H * geo.nt1();
    char *const arr = base + 4u * H * NVA;
    sfor<0, NR>([&](auto jc) {
      constexpr int j = decltype(jc)::value;
      constexpr int r = j * SPLIT + H;
      if constexpr (r < Geo::RB) {
        if (lane && geo.template live<r>()) {
          constexpr int e0 = G::row_start[r], e1 = G::row_start[r + 1];
          const __half2 o1 = u2h(st.M1[j]), od = u2h(st.M2[j]), oix = u2h(st.IX[j]);
          const uint32_t osg = st.SG[j], osg2 = st.SG2[j];
          sfor<e0, e1>([&](auto ec) {
            constexpr int e = decltype(ec)::value;
            constexpr int p = e - e0;
            if constexpr (D1 && col_deg1<G, e>()) return;
            uint32_t *tp = reinterpret_cast<uint32_t *>(arr + geo.template off<e>(i4));
            const uint32_t mag = h2u(__hfma2(__heq2(oix, u2h(h2_int<p>())), od, o1));
            *tp = h2u(__hadd2(u2h(*tp), u2h(mag ^ old_sign<p>(osg, osg2))));
          });
        }
      }
      __syncthreads();
    });
  });
  const __half2 lo = __float2half2_rn(-40.0f), hi = __float2half2_rn(40.0f);
  if (NV % 4 == 0 && NVA % 4 == 0) {
    uint4 *t4 = reinterpret_cast<uint4 *>(tot);
    for (int v = t; v < NV / 4; v += NT) {
      uint4 a = t4[v];
#pragma unroll
      for (int q = 1; q < SPLIT; ++q) {
        const uint4 o = t4[q * (NVA / 4) + v];
        a.x = h2u(__hadd2(u2h(a.x), u2h(o.x)));
        a.y = h2u(__hadd2(u2h(a.y), u2h(o.y)));
        a.z = h2u(__hadd2(u2h(a.z), u2h(o.z)));
        a.w = h2u(__hadd2(u2h(a.w), u2h(o.w)));
      }
      a.x = h2u(__hmin2(__hmax2(u2h(a.x), lo), hi));
      a.y = h2u(__hmin2(__hmax2(u2h(a.y), lo), hi));
      a.z = h2u(__hmin2(__hmax2(u2h(a.z), lo), hi));
      a.w = h2u(__hmin2(__hmax2(u2h(a.w), lo), hi));
      t4[v] = a;
    }
  } else {
    for (int v = t; v < NV; v += NT) {
      __half2 acc = u2h(tot[v]);
#pragma unroll
      for (int q = 1; q < SPLIT; ++q) acc = __hadd2(acc, u2h(tot[q * NVA + v]));
      tot[v] = h2u(__hmin2(__hmax2(acc, lo), hi));
    }
  }
  __syncthreads();
}

template <class Geo, bool ES, bool D1>
__global__ void __launch_bounds__(Geo::NT_MAX, Geo::MINB)
    k_qc_fast_h2(const QcChanParams P, const Geo geo, const float *__restrict__ llr, int64_t batch, int num_iter,
                 float alpha, int early_stop, uint8_t *__restrict__ hard_k, float *__restrict__ llr_out,
                 int32_t *__restrict__ iters_used, const uint8_t *__restrict__ ref,
                 unsigned long long *__restrict__ counts) {
  constexpr int SPLIT = Geo::SPLIT;
  extern __shared__ uint32_t smw[];
  const int NV = geo.nv(), NT = geo.nt();
  uint32_t *tot = smw;
  uint32_t *chn = smw + SPLIT * NV;
  __shared__ unsigned red[Geo::NT_MAX / 32];
  const int t = threadIdx.x;
  const int h = t / geo.nt1();
  const int i = t - h * geo.nt1();
  const bool lane = geo.full_lanes() || i < geo.z();
  char *const base = reinterpret_cast<char *>(smw);
  const int64_t cwA = 2 * (int64_t)blockIdx.x, cwB = cwA + 1;
  const bool hasB = cwB < batch;
  const float *rowA = llr + cwA * (int64_t)P.n;
  const float *rowB = hasB ? rowA + P.n : rowA;
  const __half2 al2 = __float2half2_rn(alpha);
  const bool scaled = alpha != 1.0f;
  auto chan_word = [&](int v) {
    return h2u(__floats2half2_rn(chan_value(P, rowA, v), hasB ? chan_value(P, rowB, v) : 40.0f));
  };

  for (int v = t; v < NV; v += NT) {
    const uint32_t w = chan_word(v);
    if (geo.chn_smem()) chn[v] = w;
    tot[v] = w;
  }
  H2State<Geo::NR> st;
#pragma unroll
  for (int j = 0; j < Geo::NR; ++j) st.M1[j] = st.M2[j] = st.IX[j] = st.SG[j] = st.SG2[j] = 0u;
  __syncthreads();

  int doneA = 0, doneB = hasB ? 0 : 1;
  for (int it = 0; it < num_iter; ++it) {
    const uint32_t synx = h2_cn<Geo, ES, D1>(st, base, h, lane, al2, scaled, geo,
                                             reinterpret_cast<const char *>(chn));
    if (ES && early_stop && it > 0) {
      // per-codeword syndrome of the posterior left by iteration `it`
      const int badA = __syncthreads_or(lane && ((synx >> 15) & 1u));
      const int badB = __syncthreads_or(lane && (synx >> 31));
      if (!doneA && !badA) {
        h2_emit<Geo::NT_MAX>(P, tot, NV, NT, cwA, rowA, 0, it, hard_k, llr_out, iters_used, ref, counts, red);
        doneA = 1;
      }
      if (!doneB && !badB) {
        h2_emit<Geo::NT_MAX>(P, tot, NV, NT, cwB, rowB, 1, it, hard_k, llr_out, iters_used, ref, counts, red);
        doneB = 1;
      }
      if (doneA && doneB) return;
    } else {
      __syncthreads();
    }
    h2_vn<Geo, D1>(st, tot, chn, base, h, lane, t, chan_word, geo);
  }
  if (!doneA)
    h2_emit<Geo::NT_MAX>(P, tot, NV, NT, cwA, rowA, 0, num_iter, hard_k, llr_out, iters_used, ref, counts, red);
  if (!doneB)
    h2_emit<Geo::NT_MAX>(P, tot, NV, NT, cwB, rowB, 1, num_iter, hard_k, llr_out, iters_used, ref, counts, red);
}

// first barrier step j at which slot q (rows j * SPLIT + q < RB) touches
// base column c, or -1
template <class G, int SPLIT, int RB>
__host__ __device__ constexpr int h2w_first_step(int q, int c) {
  for (int j = 0; j * SPLIT + q < RB; ++j) {
    const int r = j * SPLIT + q;
    for (int e = G::row_start[r]; e < G::row_start[r + 1]; ++e)
      if (G::col[e] == c) return j;
  }
  return -1;
}

// true when rows r1 and r2 share an accumulated (non-degree-1) column
template <class G>
__host__ __device__ constexpr bool h2w_rows_overlap(int r1, int r2) {
  for (int a = G::row_start[r1]; a < G::row_start[r1 + 1]; ++a) {
    const int c = G::col[a];
    if (G::col_start[c + 1] - G::col_start[c] == 1) continue;
    for (int b = G::row_start[r2]; b < G::row_start[r2 + 1]; ++b)
      if (G::col[b] == c) return true;
  }
  return false;
}

// Variable-node row steps of slot q: consecutive rows j, j + 1, ... that
// share no accumulated column run in one step (no barrier between them;
// every variable still receives its messages in row order).  True when slot
// q needs a barrier after its row j.
template <class G, int SPLIT, int RB>
__host__ __device__ constexpr bool h2w_step_ends(int q, int j) {
  const int r = j * SPLIT + q, rn = r + SPLIT;
  if (rn >= RB) return true;
  // the group holding row j starts at the last barrier before it
  int j0 = j;
  while (j0 > 0 && !h2w_step_ends<G, SPLIT, RB>(q, j0 - 1)) --j0;
  for (int jj = j0; jj <= j; ++jj)
    if (h2w_rows_overlap<G>(jj * SPLIT + q, rn)) return true;
  return false;
}

// Variable-node phase of the wrap-free layout (H2GeoCTW): posteriors =
// clip(chan + sum of the new messages) over the NCA accumulated columns,
// written to both copies of each column.  Both copies of T are dead once the
// check-node phase is done, so slot 0 accumulates into T's first copy, slot 1
// into its second copy and slot q >= 2 into A[q-2] (Geo::acc_word); these
// writes wrap (i + s) mod Z as usual.
template <class Geo>
__device__ __forceinline__ void h2w_vn(const H2State<Geo::NR> &st, uint32_t *smw, int h, int t) {
  using G = typename Geo::G;
  constexpr int SPLIT = Geo::SPLIT, NR = Geo::NR, Z = Geo::z(), NCA = Geo::NCA, NT = Geo::nt();
  constexpr int Z4 = Z / 4;
  static_assert(Z % 4 == 0, "wrap-free layout needs Z % 4 == 0");
  uint4 *S4w = reinterpret_cast<uint4 *>(smw);
  const uint4 *C4 = reinterpret_cast<const uint4 *>(smw + Geo::C_OFF);
  const char *Cb = reinterpret_cast<const char *>(smw + Geo::C_OFF);
  constexpr int NQ = NCA * Z4;  // uint4 words per accumulator
  // No reset pass: the first row of slot q to touch column c (in barrier-step
  // order) initialises the accumulator -- slot 0 as chan + message, slot q > 0
  // as +0 + message -- so only columns a slot never touches are reset here
  // (none for BG1 with two slots).
  constexpr bool any_untouched = [] {
    for (int q = 0; q < SPLIT; ++q)
      for (int c = 0; c < NCA; ++c)
        if (h2w_first_step<G, SPLIT, Geo::RB>(q, c) < 0) return true;
    return false;
  }();
  if constexpr (any_untouched) {
    sfor<0, NCA>([&](auto cc) {
      constexpr int c = decltype(cc)::value;
      for (int j = t; j < Z4; j += NT) {
        if constexpr (h2w_first_step<G, SPLIT, Geo::RB>(0, c) < 0) S4w[Geo::acc_word(0, c) / 4 + j] = C4[c * Z4 + j];
        sfor<1, SPLIT>([&](auto qc) {
          constexpr int q = decltype(qc)::value;
          if constexpr (h2w_first_step<G, SPLIT, Geo::RB>(q, c) < 0)
            S4w[Geo::acc_word(q, c) / 4 + j] = make_uint4(0u, 0u, 0u, 0u);
        });
      }
    });
    __syncthreads();
  }
  sfor<0, SPLIT>([&](auto hc) {
    constexpr int H = decltype(hc)::value;
    if (h != H) return;
    const unsigned i4 = 4u * tid_volatile() - 4u * H * Geo::nt1();
    char *const arr = reinterpret_cast<char *>(smw);
    sfor<0, NR>([&](auto jc) {
      constexpr int j = decltype(jc)::value;
      constexpr int r = j * SPLIT + H;
      if constexpr (r < Geo::RB) {
        constexpr int e0 = G::row_start[r], e1 = G::row_start[r + 1];
        const __half2 o1 = u2h(st.M1[j]), od = u2h(st.M2[j]), oix = u2h(st.IX[j]);
        const uint32_t osg = st.SG[j], osg2 = st.SG2[j];
        sfor<e0, e1>([&](auto ec) {
          constexpr int e = decltype(ec)::value;
          constexpr int p = e - e0;
          if constexpr (col_deg1<G, e>()) return;
          constexpr unsigned S4 = 4u * (unsigned)(G::shift[e] % Z);
          constexpr unsigned c = (unsigned)G::col[e];
          const unsigned lo4 = S4 == 0 ? i4 : min(i4 + S4, i4 + (S4 - 4u * Z));  // 4 * ((i + s) mod Z)
          uint32_t *tp = reinterpret_cast<uint32_t *>(arr + 4u * Geo::acc_word(H, (int)c) + lo4);
          const uint32_t mag = h2u(__hfma2(__heq2(oix, u2h(h2_int<p>())), od, o1));
          const __half2 msg = u2h(mag ^ old_sign<p>(osg, osg2));
          constexpr bool first = h2w_first_step<G, SPLIT, Geo::RB>(H, (int)c) == j;
          if constexpr (!first) {
            *tp = h2u(__hadd2(u2h(*tp), msg));
          } else if constexpr (H == 0) {
            const uint32_t cw = *reinterpret_cast<const uint32_t *>(Cb + 4u * Z * c + lo4);
            *tp = h2u(__hadd2(u2h(cw), msg));
          } else {
            *tp = h2u(__hadd2(u2h(0u), msg));  // +0 + m: the sum the zeroed accumulator gave
          }
        });
      }
      // the slots accumulate into disjoint arrays: each slot only waits for
      // its own warps between row steps (named barrier 1 + H), and not at all
      // between consecutive rows that share no accumulated column
      if constexpr (h2w_step_ends<G, SPLIT, Geo::RB>(H, j))
        asm volatile("bar.sync %0, %1;" ::"r"(1 + H), "r"(Geo::nt1()) : "memory");
    });
  });
  __syncthreads();
  const __half2 lo = __float2half2_rn(-40.0f), hi = __float2half2_rn(40.0f);
  auto combine = [&](int c, int j) {
    uint4 x = S4w[c * 2 * Z4 + j];
#pragma unroll
    for (int q = 1; q < SPLIT; ++q) {
      const uint4 o = S4w[(q == 1 ? c * 2 * Z4 + Z4 : Geo::T_W / 4 + (q - 2) * NQ + c * Z4) + j];
      x.x = h2u(__hadd2(u2h(x.x), u2h(o.x)));
      x.y = h2u(__hadd2(u2h(x.y), u2h(o.y)));
      x.z = h2u(__hadd2(u2h(x.z), u2h(o.z)));
      x.w = h2u(__hadd2(u2h(x.w), u2h(o.w)));
    }
    x.x = h2u(__hmin2(__hmax2(u2h(x.x), lo), hi));
    x.y = h2u(__hmin2(__hmax2(u2h(x.y), lo), hi));
    x.z = h2u(__hmin2(__hmax2(u2h(x.z), lo), hi));
    x.w = h2u(__hmin2(__hmax2(u2h(x.w), lo), hi));
    S4w[c * 2 * Z4 + j] = x;
    S4w[c * 2 * Z4 + Z4 + j] = x;
  };
  {
    if constexpr (NT % Z4 == 0) {
      // fixed (column, word) walk: no division per element
      constexpr int CS = NT / Z4;  // columns per sweep
      const int c0 = t / Z4, j = t - c0 * Z4;
#pragma unroll
      for (int c = c0; c < NCA; c += CS) combine(c, j);
    } else {
      for (int v = t; v < NQ; v += NT) {
        const int c = v / Z4;
        combine(c, v - c * Z4);
      }
    }
  }
  __syncthreads();
}

// block-wide sum of the per-thread error counts of one codeword; one bit /
// block error update (every thread calls it)
__device__ __forceinline__ void h2w_count(unsigned err, unsigned long long *counts, unsigned *red, int t, int NT) {
#pragma unroll
  for (int o = 16; o; o >>= 1) err += __shfl_xor_sync(0xffffffffu, err, o);
  if ((t & 31) == 0) red[t >> 5] = err;
  __syncthreads();
  if (t == 0) {
    unsigned long long tt = 0;
    for (int w = 0; w < NT / 32; ++w) tt += red[w];
    if (tt) {
      atomicAdd(&counts[0], tt);
      atomicAdd(&counts[1], 1ULL);
    }
  }
  __syncthreads();  // red[] is reused by the next count
}

// hard decisions of both codewords of a pair from T's first copy, 16 bits
// per thread: four 128-bit shared loads, one 128-bit store per codeword and
// the reference bits compared with one 128-bit load (k % 16 == 0, Z % 16 == 0)
template <class Geo>
__device__ __forceinline__ void h2w_emit_vec(const QcChanParams &P, const uint32_t *smw, int64_t cwA, bool hasB,
                                             int num_iter, uint8_t *hard_k, int32_t *iters_used, const uint8_t *ref,
                                             unsigned long long *counts, unsigned *red, int t) {
  constexpr int Z = Geo::z(), NT = Geo::nt();
  if (iters_used && t == 0) {
    iters_used[cwA] = num_iter;
    if (hasB) iters_used[cwA + 1] = num_iter;
  }
  unsigned errA = 0, errB = 0;
  for (int g = t; g < P.k / 16; g += NT) {
    const int v0 = 16 * g, c = v0 / Z, j = v0 - c * Z;
    uint4 rA = make_uint4(0u, 0u, 0u, 0u), rB = rA;
    if (ref) {
      rA = __ldg(reinterpret_cast<const uint4 *>(ref + cwA * (int64_t)P.k) + g);
      if (hasB) rB = __ldg(reinterpret_cast<const uint4 *>(ref + (cwA + 1) * (int64_t)P.k) + g);
    }
    const uint4 *w4 = reinterpret_cast<const uint4 *>(smw + c * 2 * Z + j);
    uint32_t ha[4], hb[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 w = w4[q];
      // (-L) > 0  <=>  L < 0 (fp16, -0 excluded): mask halves
      const uint32_t m0 = __hlt2_mask(u2h(w.x), u2h(0u)), m1 = __hlt2_mask(u2h(w.y), u2h(0u));
      const uint32_t m2 = __hlt2_mask(u2h(w.z), u2h(0u)), m3 = __hlt2_mask(u2h(w.w), u2h(0u));
      ha[q] = (m0 & 1u) | ((m1 & 1u) << 8) | ((m2 & 1u) << 16) | ((m3 & 1u) << 24);
      hb[q] = ((m0 >> 16) & 1u) | ((m1 >> 8) & 0x100u) | (m2 & 0x10000u) | ((m3 << 8) & 0x1000000u);
    }
    if (hard_k) {
      reinterpret_cast<uint4 *>(hard_k + cwA * (int64_t)P.k)[g] = make_uint4(ha[0], ha[1], ha[2], ha[3]);
      if (hasB) reinterpret_cast<uint4 *>(hard_k + (cwA + 1) * (int64_t)P.k)[g] = make_uint4(hb[0], hb[1], hb[2], hb[3]);
    }
    errA += __popc(ha[0] ^ rA.x) + __popc(ha[1] ^ rA.y) + __popc(ha[2] ^ rA.z) + __popc(ha[3] ^ rA.w);
    errB += __popc(hb[0] ^ rB.x) + __popc(hb[1] ^ rB.y) + __popc(hb[2] ^ rB.z) + __popc(hb[3] ^ rB.w);
  }
  if (ref && counts) {
    h2w_count(errA, counts, red, t, NT);
    if (hasB) h2w_count(errB, counts, red, t, NT);
  }
}

// channel words of VN v for codewords A / B, no repetition (n <= buffer):
// one load each, the same value as chan_value
__device__ __forceinline__ uint32_t chan_word_norep(const QcChanParams &P, const float *rowA, const float *rowB,
                                                    bool hasB, int v) {
  float a, b;
  if (v >= P.k && v < P.k_full) {
    a = b = 40.0f;
  } else if (v < 2 * P.z) {
    a = b = -0.0f;
  } else {
    const int pos = v < P.k ? v - 2 * P.z : P.l1 + (v - P.k_full);
    if (pos < P.n) {
      a = -(0.0f + __ldg(rowA + pos));
      b = hasB ? -(0.0f + __ldg(rowB + pos)) : 40.0f;
    } else {  // never transmitted
      a = -0.0f;
      b = hasB ? -0.0f : 40.0f;
    }
  }
  return h2u(__floats2half2_rn(a, b));
}

// Fixed-iteration fp16x2 min-sum decoder on the wrap-free layout: the
// schedule and arithmetic of k_qc_fast_h2<Geo, false, true> (bit-identical
// outputs), without the wrap arithmetic in the check-node reads.  Persistent:
// each CTA walks codeword pairs blockIdx.x, +gridDim.x, ... and prefetches
// the next pair's channel LLRs into L2 while it iterates on the current one,
// so the load at the start of a pair hits L2.  Hard decisions and counts
// only (no posterior output).
template <class Geo>
__global__ void __launch_bounds__(Geo::NT_MAX, Geo::MINB)
    k_qc_fast_h2w(const QcChanParams P, const float *__restrict__ llr, int64_t batch, int num_iter, float alpha,
                  uint8_t *__restrict__ hard_k, int32_t *__restrict__ iters_used, const uint8_t *__restrict__ ref,
                  unsigned long long *__restrict__ counts, int paths) {
  constexpr int Z = Geo::z(), NCA = Geo::NCA, NCD = Geo::NCD, NT = Geo::nt(), NVT = (NCA + NCD) * Z;
  extern __shared__ uint32_t smw[];
  uint32_t *C = smw + Geo::C_OFF;
  __shared__ unsigned red[Geo::NT_MAX / 32];
  const int t = threadIdx.x;
  const int h = t / Geo::nt1();
  const __half2 al2 = __float2half2_rn(alpha);
  const bool scaled = alpha != 1.0f;
  const bool norep = P.n <= P.buflen;
  // 16 hard decisions per thread with 128-bit loads / stores
  const bool vec_emit = P.k % 16 == 0 && Z % 16 == 0 && !(paths & 2);
  const bool vec_init = norep && Z % 4 == 0 && P.k % 4 == 0 && P.k_full % 4 == 0 && P.n % 4 == 0 && !(paths & 4);
  const int64_t npairs = (batch + 1) / 2;
  const char *base = reinterpret_cast<const char *>(smw);
  // channel word w of VN v into the layout: C (extension columns twice) and
  // both copies of T
  auto put = [&](int v, uint32_t w) {
    const int c = v / Z, j = v - c * Z;
    if (c < NCA) {
      C[v] = w;
      smw[c * 2 * Z + j] = w;
      smw[c * 2 * Z + Z + j] = w;
    } else {
      const int o = NCA * Z + (c - NCA) * 2 * Z + j;
      C[o] = w;
      C[o + Z] = w;
    }
  };
  auto prefetch_pair = [&](int64_t pr) {
    if (pr >= npairs) return;
    const int64_t cw0 = 2 * pr;
    const int64_t bytes = 4 * (int64_t)P.n * (cw0 + 1 < batch ? 2 : 1);
    const char *row = reinterpret_cast<const char *>(llr + cw0 * (int64_t)P.n);
    for (int64_t off = 128 * (int64_t)t; off < bytes; off += 128 * (int64_t)NT)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(row + off));
    if (ref) {
      const char *rr = reinterpret_cast<const char *>(ref + cw0 * (int64_t)P.k);
      const int64_t rb = (int64_t)P.k * (cw0 + 1 < batch ? 2 : 1);
      for (int64_t off = 128 * (int64_t)t; off < rb; off += 128 * (int64_t)NT)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(rr + off));
    }
  };
  prefetch_pair(blockIdx.x);
  for (int64_t pr = blockIdx.x; pr < npairs; pr += gridDim.x) {
    const int64_t cwA = 2 * pr, cwB = cwA + 1;
    const bool hasB = cwB < batch;
    const float *rowA = llr + cwA * (int64_t)P.n;
    const float *rowB = hasB ? rowA + P.n : rowA;
    if (vec_init) {
      // groups of 4 VNs (every region boundary is a multiple of 4): two
      // 128-bit loads per group, 128-bit shared stores; two groups in flight
      constexpr int NG = NVT / 4;
      for (int g0 = t; g0 < NG; g0 += 2 * NT) {
        float4 a[2], b[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int v = 4 * (g0 + u * NT);
          a[u] = b[u] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (g0 + u * NT < NG && v >= 2 * P.z && !(v >= P.k && v < P.k_full)) {
            const int pos = v < P.k ? v - 2 * P.z : P.l1 + (v - P.k_full);
            if (pos < P.n) {
              a[u] = __ldg(reinterpret_cast<const float4 *>(rowA + pos));
              if (hasB) b[u] = __ldg(reinterpret_cast<const float4 *>(rowB + pos));
            }
          }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int v = 4 * (g0 + u * NT);
          if (g0 + u * NT >= NG) continue;
          uint4 w;
          if (v >= P.k && v < P.k_full) {  // fillers: mother -40
            w.x = w.y = w.z = w.w = h2u(__float2half2_rn(40.0f));
          } else if (v < 2 * P.z) {  // punctured: +0.0
            const uint32_t z = h2u(__floats2half2_rn(-0.0f, hasB ? -0.0f : 40.0f));
            w.x = w.y = w.z = w.w = z;
          } else {  // -(0 + L), the value chan_value forms (untransmitted: -0)
            const float nb = hasB ? 0.0f : -40.0f;
            w.x = h2u(__floats2half2_rn(-(0.0f + a[u].x), -(nb + b[u].x)));
            w.y = h2u(__floats2half2_rn(-(0.0f + a[u].y), -(nb + b[u].y)));
            w.z = h2u(__floats2half2_rn(-(0.0f + a[u].z), -(nb + b[u].z)));
            w.w = h2u(__floats2half2_rn(-(0.0f + a[u].w), -(nb + b[u].w)));
          }
          const int c = v / Z, j = v - c * Z;
          if (c < NCA) {
            reinterpret_cast<uint4 *>(C)[v / 4] = w;
            reinterpret_cast<uint4 *>(smw + c * 2 * Z + j)[0] = w;
            reinterpret_cast<uint4 *>(smw + c * 2 * Z + Z + j)[0] = w;
          } else {
            const int o = NCA * Z + (c - NCA) * 2 * Z + j;
            reinterpret_cast<uint4 *>(C + o)[0] = w;
            reinterpret_cast<uint4 *>(C + o + Z)[0] = w;
          }
        }
      }
    } else if (norep) {
      // four independent loads in flight per thread
      constexpr int U = 4;
      for (int v0 = t; v0 < NVT; v0 += U * NT) {
        uint32_t w[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int v = v0 + u * NT;
          w[u] = v < NVT ? chan_word_norep(P, rowA, rowB, hasB, v) : 0u;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (v0 + u * NT < NVT) put(v0 + u * NT, w[u]);
      }
    } else {
      for (int v = t; v < NVT; v += NT)
        put(v, h2u(__floats2half2_rn(chan_value(P, rowA, v), hasB ? chan_value(P, rowB, v) : 40.0f)));
    }
    prefetch_pair(pr + gridDim.x);
    H2State<Geo::NR> st;
#pragma unroll
    for (int j = 0; j < Geo::NR; ++j) st.M1[j] = st.M2[j] = st.IX[j] = st.SG[j] = st.SG2[j] = 0u;
    __syncthreads();
    for (int it = 0; it < num_iter; ++it) {
      h2_cn<Geo, false, true>(st, base, h, true, al2, scaled, Geo{}, reinterpret_cast<const char *>(C));
      __syncthreads();
      h2w_vn<Geo>(st, smw, h, t);
    }
    // hard decisions of the systematic columns (k <= KB * Z < NCA * Z)
    if (vec_emit) {
      h2w_emit_vec<Geo>(P, smw, cwA, hasB, num_iter, hard_k, iters_used, ref, counts, red, t);
    } else {
      auto emit = [&](int64_t cw, int hb) {
        if (iters_used && t == 0) iters_used[cw] = num_iter;
        unsigned err = 0;
        for (int v = t; v < P.k; v += NT) {
          const int c = v / Z, j = v - c * Z;
          const uint32_t w = smw[c * 2 * Z + j];
          const unsigned short hv = (unsigned short)(hb ? (w >> 16) : (w & 0xFFFFu));
          const uint8_t hd = (-__half2float(__ushort_as_half(hv))) > 0.0f;
          if (hard_k) hard_k[cw * (int64_t)P.k + v] = hd;
          if (ref) err += (hd != ref[cw * (int64_t)P.k + v]);
        }
        if (ref && counts) h2w_count(err, counts, red, t, NT);
      };
      emit(cwA, 0);
      if (hasB) emit(cwB, 1);
    }
    __syncthreads();  // the next pair's channel words overwrite T
  }
}

// hard decisions of one codeword (half hb of the posterior words tot[v]),
// 16 per thread: four 128-bit shared loads, one 128-bit store, the reference
// bits compared with one 128-bit load (k % 16 == 0, 16-byte aligned rows)
__device__ __forceinline__ void h2_emit_vec1(const QcChanParams &P, const uint32_t *tot, int64_t cw, int hb, int used,
                                             uint8_t *hard_k, int32_t *iters_used, const uint8_t *ref,
                                             unsigned long long *counts, unsigned *red, int t, int NT,
                                             int colstride = 0) {
  if (iters_used && t == 0) iters_used[cw] = used;
  unsigned err = 0;
  for (int g = t; g < P.k / 16; g += NT) {
    uint4 r = make_uint4(0u, 0u, 0u, 0u);
    if (ref) r = __ldg(reinterpret_cast<const uint4 *>(ref + cw * (int64_t)P.k) + g);
    // posterior word of VN v: tot[v], or tot[(v / Z) * colstride + v % Z]
    // (16 | Z) in the wrap-free layout
    int wi = 16 * g;
    if (colstride) {
      const int c = wi / P.z;
      wi = c * colstride + (wi - c * P.z);
    }
    const uint4 *w4 = reinterpret_cast<const uint4 *>(tot + wi);
    uint32_t hv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 w = w4[q];
      uint32_t m0 = __hlt2_mask(u2h(w.x), u2h(0u)), m1 = __hlt2_mask(u2h(w.y), u2h(0u));
      uint32_t m2 = __hlt2_mask(u2h(w.z), u2h(0u)), m3 = __hlt2_mask(u2h(w.w), u2h(0u));
      if (hb) {
        m0 >>= 16;
        m1 >>= 16;
        m2 >>= 16;
        m3 >>= 16;
      }
      hv[q] = (m0 & 1u) | ((m1 & 1u) << 8) | ((m2 & 1u) << 16) | ((m3 & 1u) << 24);
    }
    if (hard_k) reinterpret_cast<uint4 *>(hard_k + cw * (int64_t)P.k)[g] = make_uint4(hv[0], hv[1], hv[2], hv[3]);
    err += __popc(hv[0] ^ r.x) + __popc(hv[1] ^ r.y) + __popc(hv[2] ^ r.z) + __popc(hv[3] ^ r.w);
  }
  if (ref && counts) h2w_count(err, counts, red, t, NT);
}

// channel words of one codeword into half q of the cached channel and
// posterior words, four VNs per 128-bit load (every region boundary a
// multiple of 4, no repetition, 16-byte aligned rows); the value chan_value
// forms
__device__ __forceinline__ void h2_refill_half_vec(const QcChanParams &P, const float *row, int q,
                                                   unsigned short *c16, unsigned short *t16, int NV, int t, int NT) {
  const int NG = NV / 4;
  for (int g0 = t; g0 < NG; g0 += 2 * NT) {
    float4 a[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int v = 4 * (g0 + u * NT);
      a[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (g0 + u * NT < NG && v >= 2 * P.z && !(v >= P.k && v < P.k_full)) {
        const int pos = v < P.k ? v - 2 * P.z : P.l1 + (v - P.k_full);
        if (pos < P.n) a[u] = __ldg(reinterpret_cast<const float4 *>(row + pos));
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int v = 4 * (g0 + u * NT);
      if (g0 + u * NT >= NG) continue;
      float f[4];
      if (v >= P.k && v < P.k_full) {
        f[0] = f[1] = f[2] = f[3] = 40.0f;
      } else if (v < 2 * P.z) {
        f[0] = f[1] = f[2] = f[3] = -0.0f;
      } else {
        f[0] = -(0.0f + a[u].x);
        f[1] = -(0.0f + a[u].y);
        f[2] = -(0.0f + a[u].z);
        f[3] = -(0.0f + a[u].w);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const unsigned short hv = __half_as_ushort(__float2half_rn(f[e]));
        c16[2 * (v + e) + q] = hv;
        t16[2 * (v + e) + q] = hv;
      }
    }
  }
}

// zero the check state of the refilled half(s): every state word keeps
// codeword A in its low and B in its high half
template <class Geo>
__device__ __forceinline__ void h2_reset_half(H2State<Geo::NR> &st, int h, int new0, int new1) {
  using G = typename Geo::G;
  constexpr int SPLIT = Geo::SPLIT, NR = Geo::NR;
  const uint32_t keep = (new0 ? 0xFFFF0000u : 0xFFFFFFFFu) & (new1 ? 0x0000FFFFu : 0xFFFFFFFFu);
  sfor<0, SPLIT>([&](auto hc) {
    constexpr int H = decltype(hc)::value;
    if (h != H) return;
    sfor<0, NR>([&](auto jc) {
      constexpr int j = decltype(jc)::value;
      constexpr int r = j * SPLIT + H;
      if constexpr (r < Geo::RB) {
        constexpr int d = G::row_start[r + 1] - G::row_start[r];
        st.M1[j] &= keep;
        st.M2[j] &= keep;
        st.IX[j] &= keep;
        st.SG[j] &= keep;
        if constexpr (d > 16) st.SG2[j] &= keep;
      }
    });
  });
}

// Persistent early-stop variant: one CTA per SM keeps two codeword slots (the
// low / high fp16 halves) busy.  When a slot's codeword converges (or reaches
// num_iter) its outputs are written and the slot is refilled with the next
// codeword from a global counter, so a converged codeword no longer idles
// while its partner keeps iterating.  Same per-codeword arithmetic and
// iteration semantics as k_qc_fast_h2 (the halves never interact).  Needs the
// channel LLRs cached in shared memory (the launcher checks).
template <class Geo, bool D1>
__global__ void __launch_bounds__(Geo::NT_MAX, 1)
    k_qc_fast_h2p(const QcChanParams P, const Geo geo, const float *__restrict__ llr, int64_t batch, int num_iter,
                  float alpha, uint8_t *__restrict__ hard_k, float *__restrict__ llr_out,
                  int32_t *__restrict__ iters_used, const uint8_t *__restrict__ ref,
                  unsigned long long *__restrict__ counts, unsigned long long *__restrict__ next, int vec) {
  constexpr int SPLIT = Geo::SPLIT;
  extern __shared__ uint32_t smw[];
  const int NV = geo.nv(), NT = geo.nt();
  uint32_t *tot = smw;
  uint32_t *chn = smw + SPLIT * NV;
  __shared__ unsigned red[Geo::NT_MAX / 32];
  __shared__ long long slot_cw[2], pend;
  __shared__ int slot_it[2], slot_new[2], pend_new;
  const int t = threadIdx.x;
  const int h = t / geo.nt1();
  const int i = t - h * geo.nt1();
  const bool lane = geo.full_lanes() || i < geo.z();
  char *const base = reinterpret_cast<char *>(smw);
  const __half2 al2 = __float2half2_rn(alpha);
  const bool scaled = alpha != 1.0f;
  H2State<Geo::NR> st;
#pragma unroll
  for (int j = 0; j < Geo::NR; ++j) st.M1[j] = st.M2[j] = st.IX[j] = st.SG[j] = st.SG2[j] = 0u;
  // codewords are claimed one ahead of need: the pending codeword's channel
  // LLRs are prefetched into L2 while the slots iterate, so a refill reads
  // them from L2 instead of waiting on HBM
  auto claim = [&]() -> long long {
    const unsigned long long c = atomicAdd(next, 1ULL);
    return (long long)c < batch ? (long long)c : -1;
  };
  if (t == 0) {
    slot_cw[0] = slot_cw[1] = -1;
    slot_it[0] = slot_it[1] = 0;
    pend = claim();
  }
  __syncthreads();
  auto chan_word = [&](int v) { return chn[v]; };  // channel words are always cached here
  for (;;) {
    // ---- refill empty slots
    if (t == 0) {
      pend_new = 0;
      for (int q = 0; q < 2; ++q) {
        slot_new[q] = 0;
        if (slot_cw[q] < 0 && pend >= 0) {
          slot_cw[q] = pend;
          slot_it[q] = 0;
          slot_new[q] = 1;
          pend = claim();
          pend_new = 1;
        }
      }
    }
    __syncthreads();
    const long long cw0 = slot_cw[0], cw1 = slot_cw[1];
    if (cw0 < 0 && cw1 < 0) return;
    const int new0 = slot_new[0], new1 = slot_new[1];
    if (pend_new && pend >= 0) {
      const char *row = reinterpret_cast<const char *>(llr + pend * (int64_t)P.n);
      for (int64_t off = 128 * (int64_t)t; off < 4 * (int64_t)P.n; off += 128 * (int64_t)NT)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(row + off));
      if (ref) {
        const char *rr = reinterpret_cast<const char *>(ref + pend * (int64_t)P.k);
        for (int off = 128 * t; off < P.k; off += 128 * NT) asm volatile("prefetch.global.L2 [%0];" ::"l"(rr + off));
      }
    }
    if (new0 | new1) {
      unsigned short *c16 = reinterpret_cast<unsigned short *>(chn);
      unsigned short *t16 = reinterpret_cast<unsigned short *>(tot);
      for (int q = 0; q < 2; ++q) {
        if (!(q ? new1 : new0)) continue;
        const float *row = llr + (q ? cw1 : cw0) * (int64_t)P.n;
        if (vec & 1) {
          h2_refill_half_vec(P, row, q, c16, t16, NV, t, NT);
        } else {
          for (int v = t; v < NV; v += NT) {
            const unsigned short hv = __half_as_ushort(__float2half_rn(chan_value(P, row, v)));
            c16[2 * v + q] = hv;
            t16[2 * v + q] = hv;
          }
        }
      }
      // fresh check state for the refilled half (the other half continues)
      h2_reset_half<Geo>(st, h, new0, new1);
      __syncthreads();
    }
    // ---- one iteration for both slots
    const uint32_t synx = h2_cn<Geo, true, D1>(st, base, h, lane, al2, scaled, geo,
                                               reinterpret_cast<const char *>(chn));
    const int bad0 = __syncthreads_or(lane && ((synx >> 15) & 1u));
    const int bad1 = __syncthreads_or(lane && (synx >> 31));
    // both_free is decided from block-uniform values only: re-reading
    // slot_cw after the barrier would race with thread 0's refill at the
    // top of the next pass
    bool freed = false, busy = false;
    for (int q = 0; q < 2; ++q) {
      const long long cw = q ? cw1 : cw0;
      if (cw < 0) continue;
      const int itq = slot_it[q];
      const bool conv = itq > 0 && !(q ? bad1 : bad0);
      busy |= !(conv || itq == num_iter);
      if (conv || itq == num_iter) {
        if (vec & 2)
          h2_emit_vec1(P, tot, cw, q, itq, hard_k, iters_used, ref, counts, red, t, NT);
        else
          h2_emit<Geo::NT_MAX>(P, tot, NV, NT, cw, llr + cw * (int64_t)P.n, q, itq, hard_k, llr_out, iters_used,
                               ref, counts, red);
        __syncthreads();
        if (t == 0) slot_cw[q] = -1;
        freed = true;
      }
    }
    if (freed) {
      __syncthreads();
      if (!busy) continue;  // both free: refill before iterating
    }
    h2_vn<Geo, D1>(st, tot, chn, base, h, lane, t, chan_word, geo);
    if (t == 0) {
      slot_it[0] += 1;
      slot_it[1] += 1;
    }
  }
}


// Persistent early-stop decoder on the wrap-free layout (H2GeoCTW): the slot
// refilling of k_qc_fast_h2p with the check-node reads, first-touch
// accumulation and combine of k_qc_fast_h2w.  Hard decisions and counts only
// (no posterior output); bit-identical to k_qc_fast_h2p<H2GeoCT, true>.
template <class Geo>
__global__ void __launch_bounds__(Geo::NT_MAX, Geo::MINB)
    k_qc_fast_h2pw(const QcChanParams P, const float *__restrict__ llr, int64_t batch, int num_iter, float alpha,
                   uint8_t *__restrict__ hard_k, int32_t *__restrict__ iters_used, const uint8_t *__restrict__ ref,
                   unsigned long long *__restrict__ counts, unsigned long long *__restrict__ next, int vec) {
  constexpr int Z = Geo::z(), NCA = Geo::NCA, NCD = Geo::NCD, NT = Geo::nt(), NVT = (NCA + NCD) * Z;
  extern __shared__ uint32_t smw[];
  uint32_t *C = smw + Geo::C_OFF;
  __shared__ unsigned red[Geo::NT_MAX / 32];
  __shared__ long long slot_cw[2], pend;
  __shared__ int slot_it[2], slot_new[2], pend_new;
  const int t = threadIdx.x;
  const int h = t / Geo::nt1();
  const char *base = reinterpret_cast<const char *>(smw);
  const __half2 al2 = __float2half2_rn(alpha);
  const bool scaled = alpha != 1.0f;
  H2State<Geo::NR> st;
#pragma unroll
  for (int j = 0; j < Geo::NR; ++j) st.M1[j] = st.M2[j] = st.IX[j] = st.SG[j] = st.SG2[j] = 0u;
  auto claim = [&]() -> long long {
    const unsigned long long c = atomicAdd(next, 1ULL);
    return (long long)c < batch ? (long long)c : -1;
  };
  if (t == 0) {
    slot_cw[0] = slot_cw[1] = -1;
    slot_it[0] = slot_it[1] = 0;
    pend = claim();
  }
  __syncthreads();
  unsigned short *c16 = reinterpret_cast<unsigned short *>(C);
  unsigned short *t16 = reinterpret_cast<unsigned short *>(smw);
  // half q of VN v's channel word into the layout (C, extension columns
  // twice, and both copies of T)
  auto put16 = [&](int v, int q, unsigned short hv) {
    const int c = v / Z, j = v - c * Z;
    if (c < NCA) {
      c16[2 * v + q] = hv;
      t16[2 * (c * 2 * Z + j) + q] = hv;
      t16[2 * (c * 2 * Z + Z + j) + q] = hv;
    } else {
      const int o = NCA * Z + (c - NCA) * 2 * Z + j;
      c16[2 * o + q] = hv;
      c16[2 * (o + Z) + q] = hv;
    }
  };
  for (;;) {
    if (t == 0) {
      pend_new = 0;
      for (int q = 0; q < 2; ++q) {
        slot_new[q] = 0;
        if (slot_cw[q] < 0 && pend >= 0) {
          slot_cw[q] = pend;
          slot_it[q] = 0;
          slot_new[q] = 1;
          pend = claim();
          pend_new = 1;
        }
      }
    }
    __syncthreads();
    const long long cw0 = slot_cw[0], cw1 = slot_cw[1];
    if (cw0 < 0 && cw1 < 0) return;
    const int new0 = slot_new[0], new1 = slot_new[1];
    if (pend_new && pend >= 0) {
      const char *row = reinterpret_cast<const char *>(llr + pend * (int64_t)P.n);
      for (int64_t off = 128 * (int64_t)t; off < 4 * (int64_t)P.n; off += 128 * (int64_t)NT)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(row + off));
      if (ref) {
        const char *rr = reinterpret_cast<const char *>(ref + pend * (int64_t)P.k);
        for (int off = 128 * t; off < P.k; off += 128 * NT) asm volatile("prefetch.global.L2 [%0];" ::"l"(rr + off));
      }
    }
    if (new0 | new1) {
      for (int q = 0; q < 2; ++q) {
        if (!(q ? new1 : new0)) continue;
        const float *row = llr + (q ? cw1 : cw0) * (int64_t)P.n;
        if (vec & 1) {
          constexpr int NG = NVT / 4;
          for (int g0 = t; g0 < NG; g0 += 2 * NT) {
            float4 a[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int v = 4 * (g0 + u * NT);
              a[u] = make_float4(0.f, 0.f, 0.f, 0.f);
              if (g0 + u * NT < NG && v >= 2 * P.z && !(v >= P.k && v < P.k_full)) {
                const int pos = v < P.k ? v - 2 * P.z : P.l1 + (v - P.k_full);
                if (pos < P.n) a[u] = __ldg(reinterpret_cast<const float4 *>(row + pos));
              }
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int v = 4 * (g0 + u * NT);
              if (g0 + u * NT >= NG) continue;
              float f[4];
              if (v >= P.k && v < P.k_full) {
                f[0] = f[1] = f[2] = f[3] = 40.0f;
              } else if (v < 2 * P.z) {
                f[0] = f[1] = f[2] = f[3] = -0.0f;
              } else {
                f[0] = -(0.0f + a[u].x);
                f[1] = -(0.0f + a[u].y);
                f[2] = -(0.0f + a[u].z);
                f[3] = -(0.0f + a[u].w);
              }
#pragma unroll
              for (int e = 0; e < 4; ++e) put16(v + e, q, __half_as_ushort(__float2half_rn(f[e])));
            }
          }
        } else {
          for (int v = t; v < NVT; v += NT) put16(v, q, __half_as_ushort(__float2half_rn(chan_value(P, row, v))));
        }
      }
      h2_reset_half<Geo>(st, h, new0, new1);
      __syncthreads();
    }
    const uint32_t synx = h2_cn<Geo, true, true>(st, base, h, true, al2, scaled, Geo{},
                                                 reinterpret_cast<const char *>(C));
    const int bad0 = __syncthreads_or((synx >> 15) & 1u);
    const int bad1 = __syncthreads_or(synx >> 31);
    // both_free is decided from block-uniform values only: re-reading
    // slot_cw after the barrier would race with thread 0's refill at the
    // top of the next pass
    bool freed = false, busy = false;
    for (int q = 0; q < 2; ++q) {
      const long long cw = q ? cw1 : cw0;
      if (cw < 0) continue;
      const int itq = slot_it[q];
      const bool conv = itq > 0 && !(q ? bad1 : bad0);
      busy |= !(conv || itq == num_iter);
      if (conv || itq == num_iter) {
        if (vec & 2) {
          h2_emit_vec1(P, smw, cw, q, itq, hard_k, iters_used, ref, counts, red, t, NT, 2 * Z);
        } else {
          if (iters_used && t == 0) iters_used[cw] = itq;
          unsigned err = 0;
          for (int v = t; v < P.k; v += NT) {
            const int c = v / Z, j = v - c * Z;
            const uint32_t w = smw[c * 2 * Z + j];
            const unsigned short hv = (unsigned short)(q ? (w >> 16) : (w & 0xFFFFu));
            const uint8_t hd = (-__half2float(__ushort_as_half(hv))) > 0.0f;
            if (hard_k) hard_k[cw * (int64_t)P.k + v] = hd;
            if (ref) err += (hd != ref[cw * (int64_t)P.k + v]);
          }
          if (ref && counts) h2w_count(err, counts, red, t, NT);
        }
        __syncthreads();
        if (t == 0) slot_cw[q] = -1;
        freed = true;
      }
    }
    if (freed) {
      __syncthreads();
      if (!busy) continue;  // both free: refill before iterating
    }
    h2w_vn<Geo>(st, smw, h, t);
    if (t == 0) {
      slot_it[0] += 1;
      slot_it[1] += 1;
    }
  }
}

// launch either kernel for a geometry with `nt` threads and `smem` bytes of
// dynamic shared memory; the persistent one when early stopping and the
// channel LLRs fit in shared memory
template <class Geo>
int launch_h2(const Geo &geo, int nt, size_t smem, bool chn_smem, const QcChanParams &P, const float *llr, int64_t B,
              int num_iter, float alpha, int early_stop, uint8_t *hard_k, float *llr_out, int32_t *iters_used,
              const uint8_t *ref, unsigned long long *counts, cudaStream_t s) {
  cudaError_t e;
  if (chn_smem && early_stop && B >= 4) {  // persistent slot-refilling decoder
    auto kp = llr_out ? k_qc_fast_h2p<Geo, false> : k_qc_fast_h2p<Geo, true>;
    e = cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_status(e, "ls_qc_decode(smem attr)");
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kp, nt, smem);
    const int64_t grid = std::min<int64_t>((int64_t)sms * std::max(1, per_sm), (B + 1) / 2);
    unsigned long long *next = nullptr;
    e = cudaMallocAsync((void **)&next, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return cuda_status(e, "ls_qc_decode(counter)");
    cudaMemsetAsync(next, 0, sizeof(unsigned long long), s);
    // 128-bit refill (bit 0) / hard-decision emit (bit 1) where the geometry
    // and the row alignment allow
    int vec = 0;
    if (P.z % 4 == 0 && P.k % 4 == 0 && P.k_full % 4 == 0 && P.n % 4 == 0 && P.n <= P.buflen &&
        !((uintptr_t)llr & 15))
      vec |= 1;
    if (!llr_out && P.k % 16 == 0 && !(((uintptr_t)hard_k | (uintptr_t)ref) & 15)) vec |= 2;
    const char *env = getenv("LSB_H2_WRAPFREE");
    if (env && env[0] == '0') vec = 0;
    kp<<<(unsigned)grid, nt, smem, s>>>(P, geo, llr, B, num_iter, alpha, hard_k, llr_out, iters_used, ref, counts,
                                        next, vec);
    e = cudaGetLastError();
    cudaFreeAsync(next, s);
    return e == cudaSuccess ? LS_OK : cuda_status(e, "ls_qc_decode");
  }
  // D1 needs the cached channel words and gives up the extension-parity
  // posteriors, so it serves fixed-iteration calls without an LLR output
  auto kern = early_stop ? k_qc_fast_h2<Geo, true, false>
                         : ((llr_out || !chn_smem) ? k_qc_fast_h2<Geo, false, false> : k_qc_fast_h2<Geo, false, true>);
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return cuda_status(e, "ls_qc_decode(smem attr)");
  const int64_t chunk = 2LL * 0x3fffffff;
  for (int64_t b0 = 0; b0 < B; b0 += chunk) {
    const int64_t nb = B - b0 < chunk ? B - b0 : chunk;
    kern<<<(unsigned)((nb + 1) / 2), nt, smem, s>>>(
        P, geo, llr + b0 * P.n, nb, num_iter, alpha, early_stop, hard_k ? hard_k + b0 * P.k : nullptr,
        llr_out ? llr_out + b0 * P.n_full : nullptr, iters_used ? iters_used + b0 : nullptr,
        ref ? ref + b0 * P.k : nullptr, counts);
  }
  e = cudaGetLastError();
  return e == cudaSuccess ? LS_OK : cuda_status(e, "ls_qc_decode");
}

// persistent wrap-free fixed-iteration decoder: one CTA per SM (or as many
// as fit), each walking codeword pairs
template <class W>
int launch_h2w(const QcChanParams &P, const float *llr, int64_t B, int num_iter, float alpha, uint8_t *hard_k,
               int32_t *iters_used, const uint8_t *ref, unsigned long long *counts, cudaStream_t s) {
  auto kern = k_qc_fast_h2w<W>;
  // the 128-bit emit (bit 2 off) and channel loads (bit 4 off) need 16-byte aligned rows
  int paths = 0;
  if (((uintptr_t)hard_k | (uintptr_t)ref) & 15) paths |= 2;
  if ((uintptr_t)llr & 15) paths |= 4;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)W::SMEM);
  if (e != cudaSuccess) return cuda_status(e, "ls_qc_decode(smem attr)");
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, W::nt(), W::SMEM);
  const int64_t grid = std::min<int64_t>((int64_t)sms * std::max(1, per_sm), (B + 1) / 2);
  if (grid > 0)
    kern<<<(unsigned)grid, W::nt(), W::SMEM, s>>>(P, llr, B, num_iter, alpha, hard_k, iters_used, ref, counts, paths);
  e = cudaGetLastError();
  return e == cudaSuccess ? LS_OK : cuda_status(e, "ls_qc_decode");
}

// persistent early-stop decoder on the wrap-free layout
template <class W>
int launch_h2pw(const QcChanParams &P, const float *llr, int64_t B, int num_iter, float alpha, uint8_t *hard_k,
                int32_t *iters_used, const uint8_t *ref, unsigned long long *counts, cudaStream_t s) {
  auto kern = k_qc_fast_h2pw<W>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)W::SMEM);
  if (e != cudaSuccess) return cuda_status(e, "ls_qc_decode(smem attr)");
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, W::nt(), W::SMEM);
  const int64_t grid = std::min<int64_t>((int64_t)sms * std::max(1, per_sm), (B + 1) / 2);
  int vec = 0;
  if (P.k % 4 == 0 && P.k_full % 4 == 0 && P.n % 4 == 0 && P.n <= P.buflen && !((uintptr_t)llr & 15)) vec |= 1;
  if (P.k % 16 == 0 && W::z() % 16 == 0 && !(((uintptr_t)hard_k | (uintptr_t)ref) & 15)) vec |= 2;
  unsigned long long *next = nullptr;
  e = cudaMallocAsync((void **)&next, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return cuda_status(e, "ls_qc_decode(counter)");
  cudaMemsetAsync(next, 0, sizeof(unsigned long long), s);
  kern<<<(unsigned)grid, W::nt(), W::SMEM, s>>>(P, llr, B, num_iter, alpha, hard_k, iters_used, ref, counts, next,
                                                 vec);
  e = cudaGetLastError();
  cudaFreeAsync(next, s);
  return e == cudaSuccess ? LS_OK : cuda_status(e, "ls_qc_decode");
}

// specialised instance (qc_instances.h)
template <class G, int Z, int R, int SPLIT>
int launch_qc_fast_h2(const QcChanParams &P, const float *llr, int64_t B, int num_iter, float alpha, int early_stop,
                      uint8_t *hard_k, float *llr_out, int32_t *iters_used, const uint8_t *ref,
                      unsigned long long *counts, cudaStream_t s) {
  using S = QcShapeH2<G, Z, R, SPLIT>;
  using W = H2GeoCTW<G, Z, R, SPLIT>;
  // fixed iterations, hard decisions only: the wrap-free layout when it fits
  // (LSB_H2_WRAPFREE=0 forces the wrapped kernel, for the bit-identity test)
  if constexpr (W::FITS && Z % 32 == 0 && R > 4) {
    const char *env = getenv("LSB_H2_WRAPFREE");
    if (!early_stop && !llr_out && S::CHN_SMEM && !(env && env[0] == '0')) {
      return launch_h2w<W>(P, llr, B, num_iter, alpha, hard_k, iters_used, ref, counts, s);
    }
    if (early_stop && !llr_out && S::CHN_SMEM && B >= 4 && !(env && env[0] == '0'))
      return launch_h2pw<W>(P, llr, B, num_iter, alpha, hard_k, iters_used, ref, counts, s);
  }
  return launch_h2(H2GeoCT<G, Z, R, SPLIT>{}, S::NT, S::SMEM, S::CHN_SMEM, P, llr, B, num_iter, alpha, early_stop,
                   hard_k, llr_out, iters_used, ref, counts, s);
}

// runtime-geometry instance: any Z <= 384 (<= 192 when SPLIT = 4) and any
// processed-row count R <= RB; `s_mod_z` are the code's shifts mod Z and
// `col` the base-graph columns, in entry order
template <class G, int RB, int SPLIT>
int launch_qc_h2rt(const QcChanParams &P, int R, const uint16_t *s_mod_z, const int32_t *col, const float *llr,
                   int64_t B, int num_iter, float alpha, int early_stop, uint8_t *hard_k, float *llr_out,
                   int32_t *iters_used, const uint8_t *ref, unsigned long long *counts, cudaStream_t s) {
  using Geo = H2GeoRT<G, RB, SPLIT>;
  static_assert(sizeof(Geo) + sizeof(QcChanParams) + 96 <= 32000, "kernel parameters too large");  // CUDA >= 12.1
  const int Z = P.z;
  if (R < 1 || R > RB) return fail(LS_EINVAL, "ls_qc_decode: row count outside the runtime-geometry instance");
  Geo geo;
  geo.Z = Z;
  geo.NT1 = ((Z + 31) / 32) * 32;
  geo.NT = geo.NT1 * SPLIT;
  if (geo.NT > Geo::NT_MAX) return fail(LS_EINVAL, "ls_qc_decode: lifting size too large for this instance");
  geo.R = R;
  geo.NV = (G::KB + (R > 4 ? R : 4)) * Z;
  geo.Z4 = 4u * (unsigned)Z;
  const size_t arr = 4 * (size_t)geo.NV;
  geo.CHN = (SPLIT + 1) * arr <= 225 * 1024;
  const size_t smem = (SPLIT + (geo.CHN ? 1 : 0)) * arr;
  if (smem > 227 * 1024) return fail(LS_EINVAL, "ls_qc_decode: code too large for the fp16x2 decoder");
  for (int e = 0; e < Geo::NE; ++e) {
    geo.s4[e] = 4u * s_mod_z[e];
    geo.cb[e] = 4u * (unsigned)Z * (unsigned)col[e];
  }
  return launch_h2(geo, geo.NT, smem, geo.CHN != 0, P, llr, B, num_iter, alpha, early_stop, hard_k, llr_out,
                   iters_used, ref, counts, s);
}

}  // namespace lsb
