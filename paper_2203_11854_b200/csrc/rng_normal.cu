// Bit-exact GPU replica of numpy's Generator.standard_normal on the
// RngStream Philox4x64-10 stream (channel.py:24-30 draws):
// the 256-level ziggurat on next_uint64, with numpy 2.3.5's tables.
//
// A normal consumes a data-dependent number of words (1 on the fast path,
// 99.2 % of draws; more on the wedge / tail paths), so draw j starts at a
// position that depends on every earlier draw.  The stream is cut into
// segments of G words and resolved in parallel:
//   1. per segment: the word lengths of every possible draw start, the rare
//      multi-word ("special") starts, and a transfer function
//        entry offset e in [0, K) -> (exit offset into the next segment,
//                                     number of draws starting in the segment)
//   2. a two-level scan composes the transfer functions (groups of segments,
//      then the groups) -> each segment's true entry offset and draw base;
//   3. per segment: every start position gets its draw index and evaluates
//      its normal.
// Only the special positions need sequential treatment, and there are ~8 of
// them per 1024 words.
#include <math.h>

#include <algorithm>

// global (L1-cached) rather than __constant__: every lane of a warp indexes
// the tables with its own random level, which the constant cache serialises
#define LS_ZIG_QUAL static __device__ const
#include "common.cuh"
#include "glibc_exp_table.h"
#include "ziggurat_tables.h"

namespace lsb {

constexpr int kZG = 1024;     // words per segment
constexpr int kZK = 32;       // entry offsets tracked per segment
constexpr int kZSpec = 96;    // max multi-word starts per segment
constexpr int kZGroup = 512;  // segments per scan group
constexpr int kZCache = 32;   // specials per segment handed from the scan pass to the emit pass

__device__ __forceinline__ uint64_t word_at(uint64_t seed, uint64_t sid, int64_t p) {
  uint64_t w[4];
  philox4x64_10((uint64_t)(p >> 2) + 1, 0, 0, 0, sid, seed, w);
  return w[p & 3];
}

__device__ __forceinline__ double dbl_at(uint64_t seed, uint64_t sid, int64_t p) {
  return (double)(word_at(seed, sid, p) >> 11) * (1.0 / 9007199254740992.0);
}

// log1p as the x86-64 glibc 2.39 libm numpy calls computes it, to the bit:
// the fdlibm argument reduction with glibc's Estrin-form polynomial and the
// exact fused-multiply-adds its FMA build contracts (checked against the host
// libm on 2e7 arguments in [-1, 0)).  This file is compiled with -fmad=false,
// so every other operation rounds separately as it does on the host.
__device__ double glibc_log1p(double x) {
  constexpr double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10,
                   two54 = 1.80143985094819840000e+16, Lp1 = 6.666666666666735130e-01,
                   Lp2 = 3.999999999940941908e-01, Lp3 = 2.857142874366239149e-01, Lp4 = 2.222219843214978396e-01,
                   Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01, Lp7 = 1.479819860511658591e-01;
  const int hx = __double2hiint(x);
  const int ax = hx & 0x7fffffff;
  double f = 0.0, c = 0.0, u;
  int k = 1, hu = 0;
  if (hx < 0x3FDA827A) {
    if (ax >= 0x3ff00000) return x == -1.0 ? -INFINITY : (x - x) / (x - x);
    if (ax < 0x3e200000) {
      if (two54 + x > 0.0 && ax < 0x3c900000) return x;
      return fma(-(x * x), 0.5, x);
    }
    if (hx > 0 || hx <= (int)0xbfd2bec3) {
      k = 0;
      f = x;
      hu = 1;
    }
  }
  if (hx >= 0x7ff00000) return x + x;
  if (k != 0) {
    if (hx < 0x43400000) {
      u = 1.0 + x;
      hu = __double2hiint(u);
      k = (hu >> 20) - 1023;
      c = (k > 0) ? 1.0 - (u - x) : x - (u - 1.0);
      c /= u;
    } else {
      u = x;
      hu = __double2hiint(u);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = __hiloint2double(hu | 0x3ff00000, __double2loint(u));
    } else {
      k += 1;
      u = __hiloint2double(hu | 0x3fe00000, __double2loint(u));
      hu = (0x00100000 - hu) >> 2;
    }
    f = u - 1.0;
  }
  const double hfsq = 0.5 * f * f, dk = (double)k;
  if (hu == 0) {
    if (f == 0.0) {
      if (k == 0) return 0.0;
      return fma(dk, ln2_hi, fma(dk, ln2_lo, c));
    }
    const double R = hfsq * fma(-0.66666666666666666, f, 1.0);
    if (k == 0) return f - R;
    return fma(dk, ln2_hi, -((R - fma(dk, ln2_lo, c)) - f));
  }
  const double s = f / (2.0 + f), z = s * s, z2 = z * z, z4 = z2 * z2, z6 = z4 * z2;
  const double R = fma(z6, fma(z, Lp7, Lp6), fma(z4, fma(z, Lp5, Lp4), fma(z, Lp1, z2 * fma(z, Lp3, Lp2))));
  if (k == 0) return f - (hfsq - (hfsq + R) * s);
  return fma(dk, ln2_hi, -((hfsq - (fma(dk, ln2_lo, c) + (hfsq + R) * s)) - f));
}

// exp(x) as the x86-64 glibc 2.39 libm numpy's ziggurat calls computes it,
// to the bit, for |x| < 512 (the wedge test's -x^2/2 lies in [-6.68, 0]):
// x = k ln2/128 + r, 2^(k/128) from glibc's table (tools/gen_glibc_exp_header.py),
// exp(r) by its degree-5 polynomial, with the fused multiply-adds of glibc's
// FMA build (checked against the host libm on 2e7 arguments in [-7, 0]).
__device__ __forceinline__ double glibc_exp(double x) {
  double kd = fma(LS_GEXP_INVLN2N, x, LS_GEXP_SHIFT);
  const uint64_t ki = (uint64_t)__double_as_longlong(kd);
  kd -= LS_GEXP_SHIFT;
  const double r = fma(kd, LS_GEXP_NEGLN2LON, fma(kd, LS_GEXP_NEGLN2HIN, x));
  const uint64_t idx = 2 * (ki % 128);
  const double tail = __longlong_as_double((long long)ls_gexp_tab[idx]);
  const uint64_t sbits = ls_gexp_tab[idx + 1] + (ki << (52 - 7));
  const double r2 = r * r;
  const double tmp = fma(r2 * r2, fma(r, LS_GEXP_C5, LS_GEXP_C4), fma(r2, fma(r, LS_GEXP_C3, LS_GEXP_C2), tail + r));
  const double scale = __longlong_as_double((long long)sbits);
  return fma(scale, tmp, scale);
}

// draw starting at word p: value and number of words consumed
__device__ double zig_draw(uint64_t seed, uint64_t sid, int64_t p, int *len) {
  const int64_t p0 = p;
  for (;;) {
    uint64_t r = word_at(seed, sid, p++);
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const int sign = (int)(r & 0x1);
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
    double x = (double)rabs * ls_zig_wi[idx];
    if (sign & 0x1) x = -x;
    if (rabs < ls_zig_ki[idx]) {
      *len = (int)(p - p0);
      return x;
    }
    if (idx == 0) {
      for (;;) {
        const double xx = -LS_ZIG_INV_R * glibc_log1p(-dbl_at(seed, sid, p++));
        const double yy = -glibc_log1p(-dbl_at(seed, sid, p++));
        if (yy + yy > xx * xx) {
          *len = (int)(p - p0);
          return ((rabs >> 8) & 0x1) ? -(LS_ZIG_R + xx) : LS_ZIG_R + xx;
        }
      }
    } else {
      const double u = dbl_at(seed, sid, p++);
      if (((ls_zig_fi[idx - 1] - ls_zig_fi[idx]) * u + ls_zig_fi[idx]) < glibc_exp(-0.5 * x * x)) {
        *len = (int)(p - p0);
        return x;
      }
    }
  }
}

// Multi-word ("special") draws of a segment, evaluated CONVERGED: the
// positions are collected first (unsorted, spos_u), then one lane per special
// walks the slow path, so a warp runs the wedge / tail code once instead of
// once per lane that happens to hold a special word.  The same lane writes its
// special at its rank (number of specials at smaller positions) into the
// position-sorted arrays: no serial sort.
__device__ __forceinline__ void zig_eval_specials(uint64_t seed, uint64_t sid, int64_t base, const uint16_t *spos_u,
                                                  uint16_t *spos, uint16_t *slen, double *sval, int n) {
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const int pk = spos_u[k];
    int len;
    const double v = zig_draw(seed, sid, base + pk, &len);
    int rank = 0;
    for (int j = 0; j < n; ++j) rank += spos_u[j] < pk;
    spos[rank] = (uint16_t)pk;
    slen[rank] = (uint16_t)min(len, 65535);
    if (sval) sval[rank] = v;
  }
}

// specials of segment s (sorted by position), shared by the segment kernels
__device__ int zig_specials(uint64_t seed, uint64_t sid, int64_t s, uint16_t *spos_u, uint16_t *spos,
                            uint16_t *slen, double *sval, int *count, int *overflow) {
  const int t = threadIdx.x;
  if (t == 0) *count = 0;
  __syncthreads();
  const int64_t base = s * kZG;
  for (int b = t; b < kZG / 4; b += blockDim.x) {
    uint64_t w[4];
    philox4x64_10((uint64_t)((base >> 2) + b) + 1, 0, 0, 0, sid, seed, w);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t r = w[u] >> 8;
      const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
      if (!(rabs < ls_zig_ki[w[u] & 0xff])) {
        const int k = atomicAdd(count, 1);
        if (k < kZSpec)
          spos_u[k] = (uint16_t)(4 * b + u);
        else
          *overflow = 1;
      }
    }
  }
  __syncthreads();
  const int n = min(*count, kZSpec);
  zig_eval_specials(seed, sid, base, spos_u, spos, slen, sval, n);
  __syncthreads();
  return n;
}

// walk the specials from entry e: number of draw starts before position `upto`
// and the next start position `cur` (>= upto means upto is not a start)
__device__ __forceinline__ void zig_walk(const uint16_t *spos, const uint16_t *slen, int n, int e, int upto,
                                         int *cnt_out, int *cur_out) {
  int cur = e, cnt = 0;
  for (int i = 0; i < n; ++i) {
    const int q = spos[i];
    if (q >= upto) break;
    if (q >= cur) {
      cnt += q - cur + 1;
      cur = q + slen[i];
    }
  }
  *cnt_out = cnt;
  *cur_out = cur;
}

// scan pass: per segment the transfer function, and the sorted specials
// (position | length << 16, value) for the emit pass, which then needs no
// slow-path draw of its own when the segment has at most kZCache of them
__global__ void k_zig_segments(uint64_t seed, uint64_t sid, int64_t nseg, uint32_t *__restrict__ trans,
                               int *__restrict__ overflow, uint32_t *__restrict__ ccnt,
                               uint32_t *__restrict__ cpl, double *__restrict__ cval) {
  __shared__ uint16_t spos_u[kZSpec], spos[kZSpec], slen[kZSpec];
  __shared__ double sval[kZSpec];
  __shared__ int count;
  for (int64_t s = blockIdx.x; s < nseg; s += gridDim.x) {
    const int n = zig_specials(seed, sid, s, spos_u, spos, slen, sval, &count, overflow);
    if (threadIdx.x == 0) ccnt[s] = (uint32_t)n;
    if ((int)threadIdx.x < n && n <= kZCache) {
      cpl[s * kZCache + threadIdx.x] = (uint32_t)spos[threadIdx.x] | ((uint32_t)slen[threadIdx.x] << 16);
      cval[s * kZCache + threadIdx.x] = sval[threadIdx.x];
    }
    const int e = threadIdx.x;
    if (e < kZK) {
      int cnt, cur;
      zig_walk(spos, slen, n, e, kZG, &cnt, &cur);
      if (cur < kZG) {
        cnt += kZG - cur;
        cur = kZG;
      }
      const int ex = cur - kZG;
      if (ex >= kZK) *overflow = 1;
      trans[s * kZK + e] = (uint32_t)cnt | ((uint32_t)min(ex, kZK - 1) << 16);
    }
    __syncthreads();
  }
}

// compose the transfer functions of each group of kZGroup segments; thread = entry
__global__ void k_zig_groups(const uint32_t *__restrict__ trans, int64_t nseg, uint32_t *__restrict__ gexit,
                             int64_t *__restrict__ gcnt) {
  const int64_t g = blockIdx.x;
  const int e = threadIdx.x;
  if (e >= kZK) return;
  int cur = e;
  int64_t tot = 0;
  const int64_t s0 = g * kZGroup, s1 = (s0 + kZGroup < nseg) ? s0 + kZGroup : nseg;
  for (int64_t s = s0; s < s1; ++s) {
    const uint32_t t = trans[s * kZK + cur];
    tot += t & 0xFFFFu;
    cur = (int)(t >> 16);
  }
  gexit[g * kZK + e] = (uint32_t)cur;
  gcnt[g * kZK + e] = tot;
}

__global__ void k_zig_top(const uint32_t *__restrict__ gexit, const int64_t *__restrict__ gcnt, int64_t ngroups,
                          int *__restrict__ gentry, int64_t *__restrict__ gbase, int64_t *__restrict__ total) {
  int cur = 0;
  int64_t base = 0;
  for (int64_t g = 0; g < ngroups; ++g) {
    gentry[g] = cur;
    gbase[g] = base;
    base += gcnt[g * kZK + cur];
    cur = (int)gexit[g * kZK + cur];
  }
  *total = base;
}

__global__ void k_zig_assign(const uint32_t *__restrict__ trans, int64_t nseg, int64_t ngroups,
                             const int *__restrict__ gentry, const int64_t *__restrict__ gbase,
                             int *__restrict__ sentry, int64_t *__restrict__ sbase) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= ngroups) return;
  int cur = gentry[g];
  int64_t base = gbase[g];
  const int64_t s0 = g * kZGroup, s1 = (s0 + kZGroup < nseg) ? s0 + kZGroup : nseg;
  for (int64_t s = s0; s < s1; ++s) {
    sentry[s] = cur;
    sbase[s] = base;
    const uint32_t t = trans[s * kZK + cur];
    base += t & 0xFFFFu;
    cur = (int)(t >> 16);
  }
}

// One block of 256 threads per segment; thread t owns the 4 words of Philox
// block t (positions 4t..4t+3), so each word is generated once: fast-path
// draws are evaluated from the registers, only the rare multi-word draws
// re-read the stream.
__global__ void __launch_bounds__(256) k_zig_emit(uint64_t seed, uint64_t sid, int64_t nseg,
                                                  const int *__restrict__ sentry, const int64_t *__restrict__ sbase,
                                                  int64_t count, double *__restrict__ out, int *__restrict__ overflow,
                                                  const uint32_t *__restrict__ ccnt, const uint32_t *__restrict__ cpl,
                                                  const double *__restrict__ cval) {
  __shared__ uint16_t spos_u[kZSpec], spos[kZSpec], slen[kZSpec];
  __shared__ double sval[kZSpec];
  __shared__ int cnt_s;
  const int t = threadIdx.x;
  for (int64_t s = blockIdx.x; s < nseg; s += gridDim.x) {
    const int64_t base = sbase[s];
    if (base >= count) continue;  // uniform per block
    if (t == 0) cnt_s = 0;
    __syncthreads();
    uint64_t w[4];
    philox4x64_10((uint64_t)(s * (kZG / 4) + t) + 1, 0, 0, 0, sid, seed, w);
    double val[4];
    uint32_t spec = 0;  // bit u: word 4t+u starts a multi-word draw
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int idx = (int)(w[u] & 0xff);
      const uint64_t r = w[u] >> 8;
      const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
      double x = (double)rabs * ls_zig_wi[idx];
      if (r & 0x1) x = -x;
      val[u] = x;
      if (!(rabs < ls_zig_ki[idx])) {
        spec |= 1u << u;
        const int k = atomicAdd(&cnt_s, 1);
        if (k < kZSpec)
          spos_u[k] = (uint16_t)(4 * t + u);
        else
          *overflow = 1;
      }
    }
    __syncthreads();
    const int n = min(cnt_s, kZSpec);
    if (ccnt[s] == (uint32_t)n && n <= kZCache) {  // handed over by the scan pass
      if (t < n) {
        const uint32_t pl = cpl[s * kZCache + t];
        spos[t] = (uint16_t)(pl & 0xFFFFu);
        slen[t] = (uint16_t)(pl >> 16);
        sval[t] = cval[s * kZCache + t];
      }
    } else {
      zig_eval_specials(seed, sid, s * kZG, spos_u, spos, slen, sval, n);
    }
    __syncthreads();
    const int e = sentry[s];
    int cnt, cur;
    zig_walk(spos, slen, n, e, 4 * t, &cnt, &cur);
    // specials of this thread, in position order, are consecutive in the list
    int k = 0;
    if (spec) {
      while (k < n && spos[k] < 4 * t) ++k;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int p = 4 * t + u;
      int len = 1;
      double v = val[u];
      if ((spec >> u) & 1u) {
        len = slen[k];
        v = sval[k];
        ++k;
      }
      if (p >= cur) {  // a draw starts here (cur >= e always)
        const int64_t j = base + cnt + (p - cur);
        if (j < count) out[j] = v;
        if (len > 1) {  // multi-word draw: the next start is p + len
          cnt += p - cur + 1;
          cur = p + len;
        }
      }
    }
    __syncthreads();
  }
}

// y = x + f32(sqrt(no/2) * z): re from normal e, im from normal S + e
// (complex_gaussian draws all real parts, then all imaginary parts)
__global__ void k_awgn_apply(const float2 *__restrict__ x, int64_t S, double scale, const double *__restrict__ z,
                             float2 *__restrict__ y) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < S; e += (int64_t)gridDim.x * blockDim.x) {
    const float2 a = x[e];
    const float nr = (float)(scale * z[e]), ni = (float)(scale * z[S + e]);
    y[e] = make_float2(a.x + nr, a.y + ni);
  }
}

// complex128 (precision "double", channel.py:27-40): noise (sqrt(no/2) * z)
// stays f64 and is added in f64
__global__ void k_awgn_apply64(const double2 *__restrict__ x, int64_t S, double scale, const double *__restrict__ z,
                               double2 *__restrict__ y) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < S; e += (int64_t)gridDim.x * blockDim.x) {
    const double2 a = x[e];
    y[e] = make_double2(a.x + scale * z[e], a.y + scale * z[S + e]);
  }
}

static int normals(uint64_t seed, uint64_t sid, int64_t count, double *out, cudaStream_t s) {
  retain_pool_memory();
  const int64_t words = (int64_t)((double)count * 1.06) + 8 * kZG;
  const int64_t nseg = (words + kZG - 1) / kZG;
  const int64_t ngroups = (nseg + kZGroup - 1) / kZGroup;
  char *ws = nullptr;
  const size_t sz_trans = sizeof(uint32_t) * nseg * kZK, sz_gx = sizeof(uint32_t) * ngroups * kZK,
               sz_gc = sizeof(int64_t) * ngroups * kZK, sz_ge = sizeof(int) * ngroups,
               sz_gb = sizeof(int64_t) * ngroups, sz_se = sizeof(int) * nseg, sz_sb = sizeof(int64_t) * nseg;
  const size_t sz_cc = sizeof(uint32_t) * nseg, sz_cp = sizeof(uint32_t) * nseg * kZCache,
               sz_cv = sizeof(double) * nseg * kZCache;
  const size_t total = sz_trans + sz_gx + sz_gc + sz_ge + sz_gb + sz_se + sz_sb + sz_cc + sz_cp + sz_cv + 160;
  cudaError_t e = cudaMallocAsync((void **)&ws, total, s);
  if (e != cudaSuccess) return cuda_status(e, "ls_standard_normal(workspace)");
  char *p = ws;
  auto take = [&](size_t n) {
    char *q = p;
    p += (n + 15) & ~size_t(15);
    return q;
  };
  uint32_t *trans = (uint32_t *)take(sz_trans);
  uint32_t *gexit = (uint32_t *)take(sz_gx);
  int64_t *gcnt = (int64_t *)take(sz_gc);
  int *gentry = (int *)take(sz_ge);
  int64_t *gbase = (int64_t *)take(sz_gb);
  int *sentry = (int *)take(sz_se);
  int64_t *sbase = (int64_t *)take(sz_sb);
  uint32_t *ccnt = (uint32_t *)take(sz_cc);
  uint32_t *cpl = (uint32_t *)take(sz_cp);
  double *cval = (double *)take(sz_cv);
  int *flags = (int *)take(16);
  int64_t *avail = (int64_t *)(flags + 2);
  cudaMemsetAsync(flags, 0, 16, s);
  const unsigned gs = (unsigned)std::min<int64_t>(nseg, 148 * 16);
  k_zig_segments<<<gs, 256, 0, s>>>(seed, sid, nseg, trans, flags, ccnt, cpl, cval);
  k_zig_groups<<<(unsigned)ngroups, kZK, 0, s>>>(trans, nseg, gexit, gcnt);
  k_zig_top<<<1, 1, 0, s>>>(gexit, gcnt, ngroups, gentry, gbase, avail);
  k_zig_assign<<<grid_for(ngroups, 128), 128, 0, s>>>(trans, nseg, ngroups, gentry, gbase, sentry, sbase);
  k_zig_emit<<<gs, 256, 0, s>>>(seed, sid, nseg, sentry, sbase, count, out, flags, ccnt, cpl, cval);
  int hflags[2] = {0, 0};
  int64_t havail = 0;
  cudaMemcpyAsync(hflags, flags, sizeof(hflags), cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&havail, avail, sizeof(havail), cudaMemcpyDeviceToHost, s);
  e = cudaStreamSynchronize(s);
  cudaFreeAsync(ws, s);
  if (e != cudaSuccess) return cuda_status(e, "ls_standard_normal");
  if (hflags[0]) return fail(LS_ECUDA, "ls_standard_normal: ziggurat segment overflow");
  if (havail < count) return fail(LS_ECUDA, "ls_standard_normal: word budget too small");
  return LS_OK;
}

}  // namespace lsb

using namespace lsb;

extern "C" int ls_standard_normal(uint64_t seed, uint64_t stream_id, int64_t count, double *out, void *stream) {
  if (count < 0 || (count && !out)) return fail(LS_EINVAL, "standard_normal: bad arguments");
  if (!count) return LS_OK;
  return normals(seed, stream_id, count, out, as_stream(stream));
}

extern "C" int ls_awgn_numpy(const float *x, int64_t count, double no, uint64_t seed, uint64_t stream_id,
                             float *y, void *stream) {
  if (no < 0) return fail(LS_EINVAL, "noise variance must be >= 0, got " + std::to_string(no));
  if (!count) return LS_OK;
  cudaStream_t s = as_stream(stream);
  if (no == 0) {
    cudaError_t e = cudaMemcpyAsync(y, x, (size_t)count * 8, cudaMemcpyDeviceToDevice, s);
    return e == cudaSuccess ? LS_OK : cuda_status(e, "ls_awgn_numpy");
  }
  double *z = nullptr;
  cudaError_t e = cudaMallocAsync((void **)&z, sizeof(double) * 2 * count, s);
  if (e != cudaSuccess) return cuda_status(e, "ls_awgn_numpy(workspace)");
  int rc = normals(seed, stream_id, 2 * count, z, s);
  if (rc == LS_OK) {
    k_awgn_apply<<<grid_for(count, 256), 256, 0, s>>>(reinterpret_cast<const float2 *>(x), count, sqrt(no / 2.0), z,
                                                      reinterpret_cast<float2 *>(y));
    e = cudaGetLastError();
    if (e != cudaSuccess) rc = cuda_status(e, "ls_awgn_numpy");
  }
  cudaFreeAsync(z, s);
  return rc;
}

extern "C" int ls_awgn_numpy64(const double *x, int64_t count, double no, uint64_t seed, uint64_t stream_id,
                               double *y, void *stream) {
  if (no < 0) return fail(LS_EINVAL, "noise variance must be >= 0, got " + std::to_string(no));
  if (!count) return LS_OK;
  cudaStream_t s = as_stream(stream);
  if (no == 0) {
    cudaError_t e = cudaMemcpyAsync(y, x, (size_t)count * 16, cudaMemcpyDeviceToDevice, s);
    return e == cudaSuccess ? LS_OK : cuda_status(e, "ls_awgn_numpy64");
  }
  double *z = nullptr;
  cudaError_t e = cudaMallocAsync((void **)&z, sizeof(double) * 2 * count, s);
  if (e != cudaSuccess) return cuda_status(e, "ls_awgn_numpy64(workspace)");
  int rc = normals(seed, stream_id, 2 * count, z, s);
  if (rc == LS_OK) {
    k_awgn_apply64<<<grid_for(count, 256), 256, 0, s>>>(reinterpret_cast<const double2 *>(x), count,
                                                        sqrt(no / 2.0), z, reinterpret_cast<double2 *>(y));
    e = cudaGetLastError();
    if (e != cudaSuccess) rc = cuda_status(e, "ls_awgn_numpy64");
  }
  cudaFreeAsync(z, s);
  return rc;
}
