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
//            phi(x) = -log(tanh(x/2)) (fp32, base 2) kept as 2^phi (ex2/rcp MUFU),
//            R = prod 2^phi = 2^S, 2^-(S - phi_e) = 2^phi_e / R,
//            c2v_new = sign * clip(phi(max(S - phi_e, 1e-12)), 0, 30) (rcp/lg2 MUFU)
//   VN phase (thread = lane j, column slot): gather + clip +-40
// Messages and posteriors are held in base-2 units (LLR * log2(e)): the phi
// arguments and results need no rescaling per edge; the channel value is
// scaled once per column and the mother LLR output once per variable.
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

// phi(x) = -log(tanh(x/2)) on the reference's clip range [1e-12, 40], in
// base-2 units: phi2(y) = phi(y ln2) / ln2 for y = x log2(e), so that
// 2^-y = e^-x.  2^phi2 = (1 + u) / (1 - u) with u = 2^-y; 1 - u comes from its
// Taylor series for small y (no cancellation).  Flush-to-zero MUFU forms (ex2,
// rcp, lg2, no denormal fix-ups): every operand here is a normal float.
constexpr float kPhiLo2 = 1e-12f * kLog2e, kClip2 = 40.0f * kLog2e;

// 1 - 2^-y without cancellation: its Taylor series for small y.  Two terms
// below y = 0.01 (truncation 8e-6 relative; 1 - u there carries the MUFU ex2
// error, ~2e-5 relative at the switch), both far below the fp16 message step.
__device__ __forceinline__ float sp_one_minus(float y, float u) {
  // 1 - 2^-y = y ln2 - (y ln2)^2 / 2 + ...
  const float series = y * fmaf(y, -kLn2 * kLn2 / 2.0f, kLn2);
  return y < 0.01f ? series : 1.0f - u;
}

// Product-domain check update (k_qc_sp): the check keeps the running product
// R = prod_e ratio_e = 2^S instead of the sum S of the per-edge phi, so the
// first phi needs no lg2 and the check no ex2 (4 MUFU per edge instead of 5).
// ratio of the clipped argument y: 2^phi2(y) = (1 + u) / (1 - u), u = 2^-y.
// The reference's upper clip (40) is not applied: above it u < 2^-57 and the
// ratio rounds to 1 either way.
__device__ __forceinline__ float sp_ratio(float y) {
  y = fmaxf(y, kPhiLo2);
  const float u = ex2_ftz(-y);
  return (1.0f + u) * rcp_ftz(sp_one_minus(y, u));
}

// phi of the exclusive sum from u = 2^-(S - phi_e) = ratio_e / R.  1 - u is
// floored at the reference's lower clip 1e-12 (ldpc.py:77-83); for a check
// whose other edges are all very reliable (1 - u below fp32 resolution) the
// message saturates near phi(1e-12) = 28.3 instead of its exact >= 17 value.
// A product past the fp32 range gives u = 0 and a zero message, the fp16
// value of the exact one (2^-S with S > 126).  The floor bounds the result
// by log2(2e12) = 40.9 (28.3 in natural units), so the reference's message
// clip at 30 (ldpc.py:143) never binds and is not applied.
__device__ __forceinline__ float sp_phi2_prod(float u) {
  return lg2_ftz((1.0f + u) * rcp_ftz(fmaxf(1.0f - u, 1e-12f)));
}

template <class G, int Z, int E>
__device__ __forceinline__ unsigned vn_off2(unsigned i2) {  // byte offset of (c, (i+s)%Z), 2-byte elements
  constexpr unsigned S2 = 2u * (unsigned)(G::shift[E] % Z);
  constexpr unsigned CB = 2u * (unsigned)Z * (unsigned)G::col[E];
  if constexpr (S2 == 0) return CB + i2;
  return CB + min(i2 + S2, i2 + (S2 - 2u * (unsigned)Z));
}

// Geometry policies (as for the fp16x2 min-sum decoder): everything
// compile-time for the specialised instances, or Z / processed rows R <= RB
// runtime with the per-edge offsets in the kernel's parameter space.
template <class G_, int Z, int R, int SPLIT_>
struct SpGeoCT {
  using G = G_;
  using S = QcShapeSP<G_, Z, R, SPLIT_>;
  static constexpr int SPLIT = SPLIT_, RB = R, NT_MAX = S::NT, MINB = S::MINB;
  static constexpr int NCOL_MAX = S::NCOL;
  __device__ __forceinline__ static constexpr int z() { return Z; }
  __device__ __forceinline__ static constexpr int nt1() { return S::NT1; }
  __device__ __forceinline__ static constexpr int nt() { return S::NT; }
  __device__ __forceinline__ static constexpr int ne() { return S::NE; }
  __device__ __forceinline__ static constexpr int ncol() { return S::NCOL; }
  __device__ __forceinline__ static constexpr bool full_lanes() { return S::NT1 == Z; }
  template <int r>
  __device__ __forceinline__ static constexpr bool live() { return true; }
  // byte offset of posterior (c, (i + s) mod Z) for lane byte offset i2
  template <int e>
  __device__ __forceinline__ static unsigned off(unsigned i2) { return vn_off2<G_, Z, e>(i2); }
  // element offset of message (e, (j - s) mod Z) for lane j
  template <int e>
  __device__ __forceinline__ static int src(int j) {
    constexpr unsigned ZS = (unsigned)(Z - G_::shift[e] % Z);  // (j - s) mod Z = (j + Z - s) mod Z
    const unsigned a = (unsigned)j + ZS;
    return e * Z + (int)min(a, a - (unsigned)Z);
  }
  template <int e>
  __device__ __forceinline__ static int ez() { return e * Z; }
};

template <class G_, int RB_, int SPLIT_>
struct SpGeoRT {
  using G = G_;
  static constexpr int SPLIT = SPLIT_, RB = RB_, NT_MAX = 768, MINB = 1;
  static constexpr int NE_MAX = G_::row_start[RB_];
  static constexpr int NCOL_MAX = G_::KB + (RB_ > 4 ? RB_ : 4);
  int Z, NT1, NT, R, NE, NCOL;
  unsigned Z2;
  uint32_t s2[NE_MAX];  // 2 * (shift mod Z)
  uint32_t cb[NE_MAX];  // 2 * Z * column
  uint32_t zs[NE_MAX];  // Z - shift mod Z
  __device__ __forceinline__ int z() const { return Z; }
  __device__ __forceinline__ int nt1() const { return NT1; }
  __device__ __forceinline__ int nt() const { return NT; }
  __device__ __forceinline__ int ne() const { return NE; }
  __device__ __forceinline__ int ncol() const { return NCOL; }
  __device__ __forceinline__ static constexpr bool full_lanes() { return false; }
  template <int r>
  __device__ __forceinline__ bool live() const { return r < R; }
  template <int e>
  __device__ __forceinline__ unsigned off(unsigned i2) const {
    const unsigned u = i2 + s2[e];
    return cb[e] + min(u, u - Z2);
  }
  template <int e>
  __device__ __forceinline__ int src(int j) const {
    const unsigned a = (unsigned)j + zs[e];
    return e * Z + (int)min(a, a - (unsigned)Z);
  }
  template <int e>
  __device__ __forceinline__ int ez() const { return e * Z; }
};

// Degree-1 shortcut (D1, fixed iterations without a posterior output): an
// extension-parity variable hears from one check only, so its message into
// that check is the channel LLR (posterior minus own message); its posterior
// stays the channel value in `tot`, its check-to-variable message is never
// formed and its column is left out of the variable update.
template <class G, int E>
__host__ __device__ constexpr bool sp_col_deg1() {
  return G::col_start[G::col[E] + 1] - G::col_start[G::col[E]] == 1;
}
template <class G, int C>
__host__ __device__ constexpr bool sp_col_is_deg1() {
  return G::col_start[C + 1] - G::col_start[C] == 1;
}

template <class Geo, bool ES, bool D1>
__global__ void __launch_bounds__(Geo::NT_MAX, Geo::MINB)
    k_qc_sp(const QcChanParams P, const Geo geo, const float *__restrict__ llr, int num_iter, int early_stop,
            uint8_t *__restrict__ hard_k, float *__restrict__ llr_out, int32_t *__restrict__ iters_used,
            const uint8_t *__restrict__ ref, unsigned long long *__restrict__ counts) {
  using G = typename Geo::G;
  constexpr int SPLIT = Geo::SPLIT;
  const int Z = geo.z(), NT = geo.nt(), NCOLZ = geo.ncol() * Z;
  extern __shared__ __half smh[];
  __half *c2v = smh;                              // [NE][Z]
  __half *tot = smh + (size_t)geo.ne() * Z;       // [NCOL][Z]
  char *const totb = reinterpret_cast<char *>(tot);
  const int t = threadIdx.x;
  const int h = t / geo.nt1();
  const int i = t - h * geo.nt1();
  const bool lane = geo.full_lanes() || i < Z;
  const int64_t b = blockIdx.x;
  const float *row = llr + b * (int64_t)P.n;

  for (int v = t; v < NCOLZ; v += NT) tot[v] = __float2half_rn(chan_value(P, row, v) * kLog2e);
  for (int q = t; q < geo.ne() * Z; q += NT) c2v[q] = __float2half_rn(0.0f);
  __syncthreads();

  int used = num_iter;
  for (int it = 0; it < num_iter; ++it) {
    // ------------------------------------------------ check-node phase
    uint32_t synx = 0;
    if (lane) {
      sfor<0, SPLIT>([&](auto hc) {
        constexpr int H = decltype(hc)::value;
        if (h != H) return;
        const unsigned i2 = 2u * (tid_volatile() - H * geo.nt1());
        const int il = (int)(i2 >> 1);
        sfor<0, (Geo::RB + SPLIT - 1) / SPLIT>([&](auto jc) {
          constexpr int r = decltype(jc)::value * SPLIT + H;
          if constexpr (r < Geo::RB) {
            if (!geo.template live<r>()) return;
            constexpr int e0 = G::row_start[r], e1 = G::row_start[r + 1], d = e1 - e0;
            float rt[d];
            uint32_t sg = 0, hs = 0;
            float rtot = 1.0f;
            sfor<e0, e1>([&](auto ec) {
              constexpr int e = decltype(ec)::value;
              constexpr int p = e - e0;
              const __half th = *reinterpret_cast<const __half *>(totb + geo.template off<e>(i2));
              if constexpr (ES) hs ^= (uint32_t)__half_as_ushort(th);
              float x = __half2float(th);
              if constexpr (!(D1 && sp_col_deg1<G, e>())) x -= __half2float(c2v[geo.template ez<e>() + il]);
              sg |= (__float_as_uint(x) >> 31) << p;
              rt[p] = sp_ratio(fabsf(x));
              rtot *= rt[p];
            });
            const uint32_t par = __popc(sg) & 1u;
            const float inv = rcp_ftz(rtot);  // 2^-S; 0 once the product overflows
            sfor<e0, e1>([&](auto ec) {
              constexpr int e = decltype(ec)::value;
              constexpr int p = e - e0;
              if constexpr (D1 && sp_col_deg1<G, e>()) return;
              const float m = sp_phi2_prod(inv * rt[p]);
              const uint32_t neg = ((par ^ (sg >> p)) & 1u) << 31;
              c2v[geo.template ez<e>() + il] = __float2half_rn(__uint_as_float(__float_as_uint(m) ^ neg));
            });
            if constexpr (ES) synx |= hs;
          }
        });
      });
    }
    if (ES && it > 0) {
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
        const int j = (int)tid_volatile() - H * geo.nt1();
        sfor<0, (Geo::NCOL_MAX + SPLIT - 1) / SPLIT>([&](auto cc) {
          constexpr int c = decltype(cc)::value * SPLIT + H;
          if constexpr (c < Geo::NCOL_MAX) {
            if constexpr (D1 && sp_col_is_deg1<G, c>()) return;
            if (c >= geo.ncol()) return;
            float sum = chan_value(P, row, c * Z + j) * kLog2e;
            constexpr int q0 = G::col_start[c], q1 = G::col_start[c + 1];
            sfor<q0, q1>([&](auto qc) {
              constexpr int e = G::col_entry[decltype(qc)::value];
              if constexpr (G::row[e] < Geo::RB) {
                if (geo.template live<G::row[e]>()) sum += __half2float(c2v[geo.template src<e>(j)]);
              }
            });
            tot[c * Z + j] = __float2half_rn(fminf(fmaxf(sum, -kClip2), kClip2));
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
    for (int v = t; v < P.n_full; v += NT) o[v] = v < NCOLZ ? -__half2float(tot[v]) * kLn2 : -chan_value(P, row, v);
  }
  unsigned err = 0;
  for (int v = t; v < P.k; v += NT) {
    const uint8_t hd = (-__half2float(tot[v])) > 0.0f;
    if (hard_k) hard_k[b * (int64_t)P.k + v] = hd;
    if (ref) err += (hd != ref[b * (int64_t)P.k + v]);
  }
  if (ref && counts) {
    __shared__ unsigned red[Geo::NT_MAX / 32];
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
  }
}

// ---------------------------------------------------------------------------
// f32-message sum-product (k_qc_sp32): the accuracy option.  Messages and
// posteriors are f32 (in base-2 units).  The first iteration reproduces the
// reference's float32 pass (ldpc.py:118-122: f32 input keeps v2c and phi in
// f32, where tanh saturates): phi from f32 tanh and log, the check sum in
// numpy's pairwise order and S - phi_e in f32.  Later iterations are f64 in
// the reference (ldpc.py:139-143); here they run in the product domain
// (sp32_msg below) with prefix/suffix products for the exclusive sets, which
// tracks the f64 log-domain result to ~1e-6 relative without its S - phi_e
// cancellation.  3 MUFU per edge; shared memory 4 * (NE + NCOL) * Z bytes, so
// it serves codes up to Z = 192 (config 3, dead rows pruned) and the small
// BG2 codes.
constexpr float kMsgClip2 = 30.0f * kLog2e;

// the reference's float32 phi of iteration 1 (natural units in, base 2 out):
// f32 tanh and log as numpy evaluates them (tanh saturates near 18).  Not
// inlined: it runs in the first iteration only, and inlining the library
// tanhf / logf at every edge of the unrolled graph would multiply the code
// size (and the instruction-cache misses of the 19 other iterations)
static __device__ __noinline__ float sp32_phi_first(float y2) {
  const float x = fminf(fmaxf(y2 * kLn2, 1e-12f), 40.0f);
  return -logf(tanhf(0.5f * x)) * kLog2e;
}

// Later iterations work in the product domain without a division or a
// cancellation: over a set of edges with u_e = 2^-y_e, N = prod (1 - u_e),
// Q = prod (1 + u_e) and P = Q - N (accumulated as P (1 + u) + 2 u N, all
// terms positive).  The log-domain sum of phi is ln(Q / N), and phi of it is
// ln((Q + N) / (Q - N)) = ln(1 + z), z = 2 N / P -- one ex2 per edge on the
// way in and one rcp + lg2 on the way out (3 MUFU per edge, the log-domain
// form needs 6).  The reference's clip of the exclusive sum to [1e-12, 40]
// (natural units) is z in [2 / (e^40 - 1), 2e12]; the message clip at 30
// never binds below that (lg2(1 + 2e12) = 28.3 nats).  lg2.approx has an
// absolute error near 2^-22, so small z takes the log1p series instead.
constexpr float kZMax = 2e12f, kZMin = 8.5e-18f;
__device__ __forceinline__ float sp32_msg(float n_ex, float p_ex) {
  const float z = fminf(fmaxf(2.0f * n_ex * rcp_ftz(p_ex), kZMin), kZMax);
  const float series =
      z * fmaf(z, fmaf(z, fmaf(z, fmaf(z, 0.2f * kLog2e, -0.25f * kLog2e), kLog2e / 3.0f), -0.5f * kLog2e), kLog2e);
  const float lg = lg2_ftz(1.0f + z);
  float r;
  asm("{\n\t.reg .pred p;\n\tsetp.lt.f32 p, %3, 0f3C800000;\n\tselp.f32 %0, %1, %2, p;\n\t}"
      : "=f"(r) : "f"(series), "f"(lg), "f"(z));
  return r;
}

template <int N>
__device__ __forceinline__ float sp32_pairwise(const float *x) {  // numpy pairwise_sum, f32
  if constexpr (N < 8) {
    float r = -0.0f;
#pragma unroll
    for (int q = 0; q < N; ++q) r = __fadd_rn(r, x[q]);
    return r;
  } else {
    float r[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) r[q] = x[q];
    constexpr int NB8 = N - N % 8;
#pragma unroll
    for (int q = 8; q < NB8; q += 8)
#pragma unroll
      for (int u = 0; u < 8; ++u) r[u] = __fadd_rn(r[u], x[q + u]);
    float res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
#pragma unroll
    for (int q = NB8; q < N; ++q) res = __fadd_rn(res, x[q]);
    return res;
  }
}

// Graph tables of the f32 kernel, built at compile time and passed by value
// (kernel parameter space): rows grouped by degree and core/extension
// columns grouped by live degree, so that one copy of a row (column) body
// per degree serves every row (column) of that degree and both thread
// groups.  Fully unrolled per-row code (260 KB) left the kernel waiting on
// instruction fetch with its 12 warps per SM (`no_instruction` 4.0 of 7.8
// cycles per issue, profiles/r02/ncu_sp32_v1_summary.txt).
template <class G, int Z, int R>
struct Sp32Tab {
  static constexpr int NE = G::row_start[R], NCOL = G::KB + (R > 4 ? R : 4);
  static constexpr int rdeg(int r) { return G::row_start[r + 1] - G::row_start[r]; }
  static constexpr int cdeg(int c) {  // entries of column c in rows < R
    int n = 0;
    for (int q = G::col_start[c]; q < G::col_start[c + 1]; ++q) n += G::row[G::col_entry[q]] < R;
    return n;
  }
  static constexpr int maxr() {
    int m = 0;
    for (int r = 0; r < R; ++r) m = rdeg(r) > m ? rdeg(r) : m;
    return m;
  }
  static constexpr int maxc() {
    int m = 0;
    for (int c = 0; c < NCOL; ++c) m = cdeg(c) > m ? cdeg(c) : m;
    return m;
  }
  static constexpr int MAXR = maxr(), MAXC = maxc();
  static constexpr bool has_rdeg(int d) {
    for (int r = 0; r < R; ++r)
      if (rdeg(r) == d) return true;
    return false;
  }
  static constexpr bool has_cdeg(int d) {
    for (int c = 0; c < NCOL; ++c)
      if (cdeg(c) == d) return true;
    return false;
  }
  uint16_t re0[R];             // first entry of each row, rows in degree order
  uint16_t roff[MAXR + 2];     // rows of degree d: re0[roff[d] .. roff[d+1])
  uint16_t ccol[NCOL];         // columns in live-degree order
  uint16_t coff[MAXC + 2];     // columns of degree d: ccol[coff[d] .. coff[d+1])
  uint16_t cst[NCOL];          // first live entry of each of them in cent
  uint2 cent[NE];              // their live entries (e * Z, Z - shift mod Z), column by column,
                               // ascending check order
  uint2 rcs[NE];               // entry e: (byte offset of its column in the posteriors, 4 * (shift mod Z))
  constexpr Sp32Tab() : re0{}, roff{}, ccol{}, coff{}, cst{}, cent{}, rcs{} {
    int k = 0;
    for (int d = 0; d <= MAXR + 1; ++d) {
      roff[d] = (uint16_t)k;
      for (int r = 0; r < R && d <= MAXR; ++r)
        if (rdeg(r) == d) re0[k++] = (uint16_t)G::row_start[r];
    }
    k = 0;
    int q = 0;
    for (int d = 0; d <= MAXC + 1; ++d) {
      coff[d] = (uint16_t)k;
      for (int c = 0; c < NCOL && d <= MAXC; ++c) {
        if (cdeg(c) != d) continue;
        cst[k] = (uint16_t)q;
        ccol[k++] = (uint16_t)c;
        for (int t = G::col_start[c]; t < G::col_start[c + 1]; ++t) {
          const int e = G::col_entry[t];
          if (G::row[e] < R) cent[q++] = uint2{(uint32_t)(e * Z), (uint32_t)(Z - G::shift[e] % Z)};
        }
      }
    }
    for (int e = 0; e < NE; ++e)
      rcs[e] = uint2{4u * (uint32_t)Z * (uint32_t)G::col[e], 4u * (uint32_t)(G::shift[e] % Z)};
  }
};

// GM: the f32 messages do not fit in shared memory with the posteriors
// (config 2: 344 KB); they live in an L2-resident slice per CTA and the
// CTAs loop over the batch (persistent grid)
template <class G, int Z, int R, int SPLIT, bool ES, bool GM>
__global__ void __launch_bounds__(QcShapeSP<G, Z, R, SPLIT>::NT, GM ? 2 : QcShapeSP<G, Z, R, SPLIT>::MINB)
    k_qc_sp32(const QcChanParams P, const Sp32Tab<G, Z, R> tab, const float *__restrict__ llr, int64_t batch,
              int num_iter, uint8_t *__restrict__ hard_k, float *__restrict__ llr_out,
              int32_t *__restrict__ iters_used, const uint8_t *__restrict__ ref, unsigned long long *__restrict__ counts,
              float *__restrict__ c2vws) {
  using S = QcShapeSP<G, Z, R, SPLIT>;
  using Tab = Sp32Tab<G, Z, R>;
  constexpr int NT = S::NT, NT1 = S::NT1, NCOLZ = S::NCOL * Z;
  extern __shared__ float smf[];
  float *c2v = GM ? c2vws + (size_t)blockIdx.x * S::NE * Z : smf;  // [NE][Z]
  float *tot = GM ? smf : smf + (size_t)S::NE * Z;                   // [NCOL][Z]
  const char *const totb = reinterpret_cast<const char *>(tot);
  const int t = threadIdx.x;
  const int h = t / NT1;  // thread group: every SPLIT-th row / column of each degree class
  const int i = t - h * NT1;
  const bool lane = NT1 == Z || i < Z;
  for (int64_t b = blockIdx.x; b < batch; b += gridDim.x) {
  const float *row = llr + b * (int64_t)P.n;

  for (int v = t; v < NCOLZ; v += NT) tot[v] = chan_value(P, row, v) * kLog2e;
  for (int q = t; q < S::NE * Z; q += NT) c2v[q] = 0.0f;
  __syncthreads();

  // one check-node phase; FIRST = the reference's float32 first pass
  auto cn_phase = [&](auto first_c) -> uint32_t {
    constexpr bool first = decltype(first_c)::value;
    uint32_t synx = 0;
    if (lane) {
      uint32_t i4 = 4u * (uint32_t)i;
      asm volatile("" : "+r"(i4));
      sfor<1, Tab::MAXR + 1>([&](auto dc) {
        constexpr int d = decltype(dc)::value;
        if constexpr (Tab::has_rdeg(d)) {
          for (int rr = tab.roff[d] + h; rr < tab.roff[d + 1]; rr += SPLIT) {
            const int e0 = tab.re0[rr];
            float ph[first ? d : 1], uu[first ? 1 : d], nn[first ? 1 : d], pn[first ? 1 : d], pp[first ? 1 : d];
            float na = 1.0f, pa = 0.0f;
            uint32_t sg = 0, hs = 0;
#pragma unroll
            for (int p = 0; p < d; ++p) {
              const int e = e0 + p;
              const uint2 cs = tab.rcs[e];
              uint32_t o = i4 + cs.y;
              o = min(o, o - 4u * Z);
              const float tv = *reinterpret_cast<const float *>(totb + cs.x + o);
              if constexpr (ES) hs ^= __float_as_uint(tv);
              const float x = tv - c2v[e * Z + i];
              sg |= (__float_as_uint(x) >> 31) << p;
              if constexpr (first) {
                ph[p] = sp32_phi_first(fabsf(x));
              } else {
                const float y = fminf(fmaxf(fabsf(x), kPhiLo2), kClip2);
                const float u = ex2_ftz(-y);
                uu[p] = u;
                nn[p] = sp_one_minus(y, u);
                pn[p] = na;
                pp[p] = pa;
                // (N, P) <- (N (1 - u), P (1 + u) + 2 u N): Q = N + P stays implicit
                pa = fmaf(2.0f * u, na, fmaf(pa, u, pa));
                na *= nn[p];
              }
            }
            const uint32_t par = __popc(sg) & 1u;
            if constexpr (first) {  // the reference's f32 pass: psum in pairwise order, then psum - pmag
              const float ps = __fadd_rn(ph[0], sp32_pairwise<d - 1>(ph + 1));
#pragma unroll
              for (int p = 0; p < d; ++p) {
                const float m = fminf(sp32_phi_first(__fsub_rn(ps, ph[p])), kMsgClip2);
                const uint32_t neg = ((par ^ (sg >> p)) & 1u) << 31;
                c2v[(e0 + p) * Z + i] = __uint_as_float(__float_as_uint(m) ^ neg);
              }
            } else {
              // exclusive (N, P) of every edge from the prefix (pn, pp) and a
              // running suffix (nb, pb): N_ex = N_a N_b, P_ex = P_a Q_b + N_a P_b
              float nb = 1.0f, pb = 0.0f;
#pragma unroll
              for (int p = d - 1; p >= 0; --p) {
                const float m = sp32_msg(pn[p] * nb, fmaf(pp[p], nb + pb, pn[p] * pb));
                const uint32_t neg = ((par ^ (sg >> p)) & 1u) << 31;
                c2v[(e0 + p) * Z + i] = __uint_as_float(__float_as_uint(m) ^ neg);
                pb = fmaf(2.0f * uu[p], nb, fmaf(pb, uu[p], pb));
                nb *= nn[p];
              }
            }
            if constexpr (ES) synx |= hs;
          }
        }
      });
    }
    return synx;
  };

  int used = num_iter;
  for (int it = 0; it < num_iter; ++it) {
    const uint32_t synx = it == 0 ? cn_phase(std::true_type{}) : cn_phase(std::false_type{});
    if (ES && it > 0) {
      if (!__syncthreads_or(lane && (synx >> 31))) {
        used = it;
        break;
      }
    } else {
      __syncthreads();
    }
    // ------------------------------------------------ variable-node phase (gather)
    if (lane) {
      const int j = i;
      sfor<1, Tab::MAXC + 1>([&](auto dc) {
        constexpr int d = decltype(dc)::value;
        if constexpr (Tab::has_cdeg(d)) {
          for (int cc = tab.coff[d] + h; cc < tab.coff[d + 1]; cc += SPLIT) {
            const int c = tab.ccol[cc];
            const int q0 = tab.cst[cc];
            float sum = chan_value(P, row, c * Z + j) * kLog2e;
#pragma unroll
            for (int q = 0; q < d; ++q) {
              const uint2 ez = tab.cent[q0 + q];
              const unsigned a = (unsigned)j + ez.y;
              sum += c2v[ez.x + min(a, a - (unsigned)Z)];
            }
            tot[c * Z + j] = fminf(fmaxf(sum, -kClip2), kClip2);
          }
        }
      });
    }
    __syncthreads();
  }

  if (iters_used && t == 0) iters_used[b] = used;
  if (llr_out) {
    float *o = llr_out + b * (int64_t)P.n_full;
    for (int v = t; v < P.n_full; v += NT) o[v] = v < NCOLZ ? -tot[v] * kLn2 : -chan_value(P, row, v);
  }
  unsigned err = 0;
  for (int v = t; v < P.k; v += NT) {
    const uint8_t hd = (-tot[v]) > 0.0f;
    if (hard_k) hard_k[b * (int64_t)P.k + v] = hd;
    if (ref) err += (hd != ref[b * (int64_t)P.k + v]);
  }
  if (ref && counts) {
    __shared__ unsigned red[NT / 32];
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
  }
  __syncthreads();
  }
}

template <class G, int Z, int R, int SPLIT>
int launch_qc_sp32(const QcChanParams &P, const float *llr, int64_t B, int num_iter, float alpha, int early_stop,
                   uint8_t *hard_k, float *llr_out, int32_t *iters_used, const uint8_t *ref,
                   unsigned long long *counts, cudaStream_t s) {
  (void)alpha;
  using S = QcShapeSP<G, Z, R, SPLIT>;
  using Tab = Sp32Tab<G, Z, R>;
  static_assert(sizeof(Tab) + sizeof(QcChanParams) + 128 <= 32000, "kernel parameters too large");
  // f32 messages and posteriors in shared memory, or the messages in L2
  constexpr bool GM = 2 * S::SMEM > 227 * 1024;
  constexpr size_t smem = GM ? 4ull * S::NCOL * Z : 2 * S::SMEM;
  static_assert(smem <= 227 * 1024, "f32 sum-product posteriors do not fit in shared memory");
  static constexpr Tab tab{};
  auto kern = early_stop ? k_qc_sp32<G, Z, R, SPLIT, true, GM> : k_qc_sp32<G, Z, R, SPLIT, false, GM>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return cuda_status(e, "ls_qc_decode(smem attr)");
  if (B <= 0) return LS_OK;
  float *ws = nullptr;
  int64_t grid = B;
  if (GM) {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, S::NT, smem);
    grid = std::min<int64_t>((int64_t)sms * std::max(1, per_sm), B);
    retain_pool_memory();
    e = cudaMallocAsync((void **)&ws, sizeof(float) * (size_t)grid * S::NE * Z, s);
    if (e != cudaSuccess) return cuda_status(e, "ls_qc_decode(sp32 message workspace)");
  }
  for (int64_t b0 = 0; b0 < B; b0 += 0x7fffffff) {
    const int64_t nb = B - b0 < 0x7fffffff ? B - b0 : 0x7fffffff;
    const int64_t g = std::min<int64_t>(grid, nb);
    kern<<<(unsigned)g, S::NT, smem, s>>>(P, tab, llr + b0 * P.n, nb, num_iter, hard_k ? hard_k + b0 * P.k : nullptr,
                                          llr_out ? llr_out + b0 * P.n_full : nullptr,
                                          iters_used ? iters_used + b0 : nullptr, ref ? ref + b0 * P.k : nullptr,
                                          counts, ws);
  }
  e = cudaGetLastError();
  if (ws) cudaFreeAsync(ws, s);
  return e == cudaSuccess ? LS_OK : cuda_status(e, "ls_qc_decode");
}

template <class Geo>
int launch_sp(const Geo &geo, int nt, size_t smem, const QcChanParams &P, const float *llr, int64_t B,
              int num_iter, int early_stop, uint8_t *hard_k, float *llr_out, int32_t *iters_used,
              const uint8_t *ref, unsigned long long *counts, cudaStream_t s) {
  auto kern = early_stop ? k_qc_sp<Geo, true, false> : (llr_out ? k_qc_sp<Geo, false, false> : k_qc_sp<Geo, false, true>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return cuda_status(e, "ls_qc_decode(smem attr)");
  for (int64_t b0 = 0; b0 < B; b0 += 0x7fffffff) {
    const int64_t nb = B - b0 < 0x7fffffff ? B - b0 : 0x7fffffff;
    kern<<<(unsigned)nb, nt, smem, s>>>(P, geo, llr + b0 * P.n, num_iter, early_stop,
                                        hard_k ? hard_k + b0 * P.k : nullptr,
                                        llr_out ? llr_out + b0 * P.n_full : nullptr,
                                        iters_used ? iters_used + b0 : nullptr, ref ? ref + b0 * P.k : nullptr,
                                        counts);
  }
  e = cudaGetLastError();
  return e == cudaSuccess ? LS_OK : cuda_status(e, "ls_qc_decode");
}

template <class G, int Z, int R, int SPLIT>
int launch_qc_sp(const QcChanParams &P, const float *llr, int64_t B, int num_iter, float alpha, int early_stop,
                 uint8_t *hard_k, float *llr_out, int32_t *iters_used, const uint8_t *ref,
                 unsigned long long *counts, cudaStream_t s) {
  (void)alpha;
  using S = QcShapeSP<G, Z, R, SPLIT>;
  static_assert(S::SMEM <= 227 * 1024, "sum-product messages do not fit in shared memory");
  return launch_sp(SpGeoCT<G, Z, R, SPLIT>{}, S::NT, S::SMEM, P, llr, B, num_iter, early_stop, hard_k, llr_out,
                   iters_used, ref, counts, s);
}

// runtime-geometry sum-product instance: any Z with NT1 * SPLIT <= 768 and any
// R <= RB whose messages fit in shared memory
template <class G, int RB, int SPLIT>
int launch_qc_sprt(const QcChanParams &P, int R, const uint16_t *s_mod_z, const int32_t *col, const float *llr,
                   int64_t B, int num_iter, float alpha, int early_stop, uint8_t *hard_k, float *llr_out,
                   int32_t *iters_used, const uint8_t *ref, unsigned long long *counts, cudaStream_t s) {
  (void)alpha;
  using Geo = SpGeoRT<G, RB, SPLIT>;
  static_assert(sizeof(Geo) + sizeof(QcChanParams) + 96 <= 32000, "kernel parameters too large");
  const int Z = P.z;
  if (R < 1 || R > RB) return fail(LS_EINVAL, "ls_qc_decode: row count outside the runtime-geometry instance");
  Geo geo;
  geo.Z = Z;
  geo.NT1 = ((Z + 31) / 32) * 32;
  geo.NT = geo.NT1 * SPLIT;
  if (geo.NT > Geo::NT_MAX) return fail(LS_EINVAL, "ls_qc_decode: lifting size too large for this instance");
  geo.R = R;
  geo.NE = G::row_start[R];
  geo.NCOL = G::KB + (R > 4 ? R : 4);
  geo.Z2 = 2u * (unsigned)Z;
  const size_t smem = 2ull * ((size_t)geo.NE * Z + (size_t)geo.NCOL * Z);
  if (smem > 227 * 1024)
    return fail(LS_EINVAL, "ls_qc_decode: sum-product messages of this code do not fit in shared memory; "
                           "use the exact decoder");
  for (int e = 0; e < Geo::NE_MAX; ++e) {
    geo.s2[e] = 2u * s_mod_z[e];
    geo.cb[e] = 2u * (unsigned)Z * (unsigned)col[e];
    geo.zs[e] = (unsigned)(Z - s_mod_z[e]);
  }
  return launch_sp(geo, geo.NT, smem, P, llr, B, num_iter, early_stop, hard_k, llr_out, iters_used, ref, counts,
                   s);
}

}  // namespace lsb
