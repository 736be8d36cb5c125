// C-ABI glue: errors, code/graph handles, and the streaming kernels of the
// chain (source, mapper, AWGN, demapper, encoder, derate, error counting).
// Decoders live in bp_exact.cu and bp_fast.cu.
#include <math.h>
#include <stdio.h>

#include <algorithm>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace lsb {

static thread_local std::string g_err;

void retain_pool_memory() {
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  });
}

void set_error(const std::string &msg) { g_err = msg; }
int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}
int cuda_status(cudaError_t e, const char *where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return LS_ECUDA;
}

// ------------------------------------------------------------ binary_source
// One thread per Philox block = 4 uint64 words = 32 payload bits.  Bit j of
// word w is (w >> (8j+7)) & 1: low uint32 half first, bytes LSB first, each
// bit the byte's MSB (numpy bounded uint8 draw).
// `blk0` = index of the first Philox block (32 bits each) of this slice of
// the stream, so a [B, k] draw can be produced in row chunks.
__global__ void k_binary_source(uint64_t seed, uint64_t sid, int64_t blk0, int64_t count,
                                uint8_t *__restrict__ bits) {
  const int64_t nblk = (count + 31) / 32;
  for (int64_t blk = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; blk < nblk;
       blk += (int64_t)gridDim.x * blockDim.x) {
    uint64_t w[4];
    philox4x64_10((uint64_t)(blk0 + blk) + 1, 0, 0, 0, sid, seed, w);
    const int64_t base = blk * 32;
    if (base + 32 <= count && ((reinterpret_cast<uintptr_t>(bits + base) & 15) == 0)) {
      uint32_t o[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        uint64_t word = w[q / 2];
        uint32_t v = 0;
#pragma unroll
        for (int t = 0; t < 4; ++t) v |= (uint32_t)((word >> (8 * (4 * (q % 2) + t) + 7)) & 1) << (8 * t);
        o[q] = v;
      }
      uint4 *dst = reinterpret_cast<uint4 *>(bits + base);
      dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
      dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
    } else {
      for (int j = 0; j < 32 && base + j < count; ++j)
        bits[base + j] = (uint8_t)((w[j / 8] >> (8 * (j % 8) + 7)) & 1);
    }
  }
}

// ------------------------------------------------------------ map_bits
__global__ void k_map_bits(const uint8_t *__restrict__ bits, int64_t nsym, int m,
                           const float2 *__restrict__ pts, float2 *__restrict__ x) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nsym;
       s += (int64_t)gridDim.x * blockDim.x) {
    int lab = 0;
    for (int t = 0; t < m; ++t) lab = (lab << 1) | (bits[s * m + t] & 1);
    x[s] = pts[lab];
  }
}

// complex128 points (precision "double": the reference keeps map_bits' f64
// points, sweep.py:170, 352)
__global__ void k_map_bits64(const uint8_t *__restrict__ bits, int64_t nsym, int m,
                             const double2 *__restrict__ pts, double2 *__restrict__ x) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nsym;
       s += (int64_t)gridDim.x * blockDim.x) {
    int lab = 0;
    for (int t = 0; t < m; ++t) lab = (lab << 1) | (bits[s * m + t] & 1);
    x[s] = pts[lab];
  }
}

// ------------------------------------------------------------ awgn (fast mode)
// Counter-based: element pair q uses Philox4x32 counter (q, stream lo, stream hi, 0)
// under key (seed lo, seed hi); Box-Muller gives two complex normals per call.
// standard complex normals (unit variance per real component) for complex
// elements 2q and 2q+1 of stream (seed, sid)
__device__ __forceinline__ void normal_pair(int64_t q, uint64_t seed, uint64_t sid, float2 &n0, float2 &n1) {
  uint4 r = philox4x32_10(make_uint4((uint32_t)q, (uint32_t)(q >> 32), (uint32_t)sid, (uint32_t)(sid >> 32)),
                          make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
  // Box-Muller on uniforms u in (0,1] (radius) and angles in [-pi, pi):
  // rad = sqrt(-2 ln u) = sqrt(-2 ln2 log2 u); one SFU op each for the log,
  // the square root, the sine and the cosine
  constexpr float k24 = 1.0f / 16777216.0f, kTwoPi24 = 6.283185307179586f / 16777216.0f;
  const float u0 = (float)((r.x >> 8) + 1) * k24, u2 = (float)((r.z >> 8) + 1) * k24;
  const float a1 = fmaf((float)(r.y >> 8), kTwoPi24, -3.14159265358979f);
  const float a3 = fmaf((float)(r.w >> 8), kTwoPi24, -3.14159265358979f);
  const float rad0 = sqrt_ftz(-2.0f * kLn2 * lg2_ftz(u0)), rad1 = sqrt_ftz(-2.0f * kLn2 * lg2_ftz(u2));
  n0 = make_float2(rad0 * cos_ftz(a1), rad0 * sin_ftz(a1));
  n1 = make_float2(rad1 * cos_ftz(a3), rad1 * sin_ftz(a3));
}

__global__ void k_awgn(const float2 *__restrict__ x, int64_t count, float sigma, uint64_t seed,
                       uint64_t sid, int64_t q0, float2 *__restrict__ y) {
  const int64_t npair = (count + 1) / 2;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < npair;
       q += (int64_t)gridDim.x * blockDim.x) {
    float2 n0, n1;
    normal_pair(q0 + q, seed, sid, n0, n1);
    int64_t e0 = 2 * q;
    float2 a = x[e0];
    y[e0] = make_float2(a.x + sigma * n0.x, a.y + sigma * n0.y);
    if (e0 + 1 < count) {
      float2 b = x[e0 + 1];
      y[e0 + 1] = make_float2(b.x + sigma * n1.x, b.y + sigma * n1.y);
    }
  }
}

// Fused map_bits -> awgn -> demap for Gray QAM (the Pipeline's fast chain):
// coded bits [nsym*m] in, f32 LLRs [nsym*m] out, no symbol arrays in HBM.
// Same points, noise stream and arithmetic order as k_map_bits + k_awgn
// (y is bit-identical); the per-axis log-sum-exp runs in f32, base 2, on the
// SFU (ex2 / lg2; |dLLR| ~1e-6 against the f64 demapper, inside the 1e-4
// tolerance).
struct QamAxesF {
  float amp[16];
  int lab[16];
};

template <int HALF, bool VEC>
__global__ void k_modem_qam(const uint8_t *__restrict__ bits, int64_t nsym, const float2 *__restrict__ pts,
                            float sigma, float inv_no, uint64_t seed, uint64_t sid, int64_t q0, const QamAxesF A,
                            int maxlog, float *__restrict__ llr) {
  constexpr int L = 1 << HALF, M = 2 * HALF;
  const float inv_no2 = inv_no * kLog2e;
  __shared__ float s_amp[L];
  __shared__ float2 s_pts[L * L];
  if (threadIdx.x < L) s_amp[threadIdx.x] = A.amp[threadIdx.x];
  for (int p = threadIdx.x; p < L * L; p += blockDim.x) s_pts[p] = pts[p];
  __syncthreads();
  const int64_t npair = (nsym + 1) / 2;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < npair;
       q += (int64_t)gridDim.x * blockDim.x) {
    float2 nz[2];
    normal_pair(q0 + q, seed, sid, nz[0], nz[1]);
    // VEC: the pair's 2M bit bytes in M/2 32-bit loads and its 2M LLRs in
    // M/2 16-byte stores (full pairs only; needs 4-byte aligned bits and
    // 16-byte aligned LLRs)
    const bool full = VEC && 2 * q + 1 < nsym;
    uint32_t w[VEC ? M / 2 : 1];
    if (full) {
      const uint32_t *b4 = reinterpret_cast<const uint32_t *>(bits + 2 * q * M);
#pragma unroll
      for (int k = 0; k < (VEC ? M / 2 : 1); ++k) w[k] = b4[k];
    }
    float out[2][M];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t s = 2 * q + u;
      if (s >= nsym) break;
      int label = 0;
#pragma unroll
      for (int t = 0; t < M; ++t) {
        const int bi = u * M + t;
        const uint32_t bt = full ? (w[bi >> 2] >> (8 * (bi & 3))) : bits[s * M + t];
        label = (label << 1) | (bt & 1);
      }
      const float2 x = s_pts[label];
      const float yv[2] = {x.x + sigma * nz[u].x, x.y + sigma * nz[u].y};
#pragma unroll
      for (int ax = 0; ax < 2; ++ax) {
        float lg[L];  // logits in base-2 units
        float top = -INFINITY;
#pragma unroll
        for (int l = 0; l < L; ++l) {
          const float d = yv[ax] - s_amp[l];
          lg[l] = -(d * d) * inv_no2;
          top = fmaxf(top, lg[l]);
        }
        // APP: one exponential per level against the axis maximum, shared by
        // the axis's bits (L instead of L * HALF SFU exponentials); the subset
        // holding the maximum sums to >= 1, the other can only underflow when
        // its log-sum is more than 126 below, where max-log is exact
        float ex[L];
        if (!maxlog) {
#pragma unroll
          for (int l = 0; l < L; ++l) ex[l] = ex2_ftz(lg[l] - top);
        }
#pragma unroll
        for (int t = 0; t < HALF; ++t) {
          const int sh = HALF - 1 - t;
          float mx1 = -INFINITY, mx0 = -INFINITY, s1 = 0.0f, s0 = 0.0f;
#pragma unroll
          for (int l = 0; l < L; ++l) {  // level l carries Gray label l ^ (l >> 1)
            if (((l ^ (l >> 1)) >> sh) & 1) {
              mx1 = fmaxf(mx1, lg[l]);
              if (!maxlog) s1 += ex[l];
            } else {
              mx0 = fmaxf(mx0, lg[l]);
              if (!maxlog) s0 += ex[l];
            }
          }
          float v = mx1 - mx0;
          if (!maxlog && s1 > 0.0f && s0 > 0.0f) v = lg2_ftz(s1) - lg2_ftz(s0);
          out[u][2 * t + ax] = v * kLn2;
        }
      }
      if (!full) {
#pragma unroll
        for (int j = 0; j < M; ++j) llr[s * M + j] = out[u][j];
      }
    }
    if (full) {
      float4 *o4 = reinterpret_cast<float4 *>(llr + 2 * q * M);
#pragma unroll
      for (int k = 0; k < (VEC ? M / 2 : 1); ++k) {
        const int j = 4 * k;
        o4[k] = make_float4(out[j / M][j % M], out[(j + 1) / M][(j + 1) % M], out[(j + 2) / M][(j + 2) % M],
                            out[(j + 3) / M][(j + 3) % M]);
      }
    }
  }
}

// ------------------------------------------------------------ demapper
// received symbol s as (re, im) in f64: complex64 input is upcast as numpy
// does (mapping.py:120), complex128 read as is
__device__ __forceinline__ double2 ld_sym(const float2 *__restrict__ y, int64_t s) {
  const float2 v = y[s];
  return make_double2((double)v.x, (double)v.y);
}
__device__ __forceinline__ double2 ld_sym(const double2 *__restrict__ y, int64_t s) { return y[s]; }

// mapping.py:110-143: logits = -|y - p|^2 / no (f64), LLR_j = LSE(bit_j=1) -
// LSE(bit_j=0) with scipy's max + log1p(sum of the others), or max - max.
template <int MAXP, class YT>
__global__ void k_demap(const YT *__restrict__ y, int64_t nsym, double no,
                        const double *__restrict__ no_vec, const double *__restrict__ prior,
                        const double2 *__restrict__ pts, int m, int mode, float *__restrict__ llr32,
                        double *__restrict__ llr64) {
  const int P = 1 << m;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nsym;
       s += (int64_t)gridDim.x * blockDim.x) {
    const double2 ys = ld_sym(y, s);
    const double yr = ys.x, yi = ys.y;
    const double nos = no_vec ? no_vec[s] : no;
    double lg[MAXP];
    for (int p = 0; p < P; ++p) {
      double dr = yr - pts[p].x, di = yi - pts[p].y;
      double h = hypot(dr, di);
      lg[p] = -(h * h) / nos;
      if (prior) {  // + bits(p) . prior (mapping.py:123-131)
        double pr = 0.0;
        for (int j = 0; j < m; ++j)
          if ((p >> (m - 1 - j)) & 1) pr += prior[s * m + j];
        lg[p] += pr;
      }
    }
    for (int j = 0; j < m; ++j) {
      const int sh = m - 1 - j;
      double mx1 = -INFINITY, mx0 = -INFINITY;
      int a1 = -1, a0 = -1;
      for (int p = 0; p < P; ++p) {
        if ((p >> sh) & 1) {
          if (lg[p] > mx1) { mx1 = lg[p]; a1 = p; }
        } else {
          if (lg[p] > mx0) { mx0 = lg[p]; a0 = p; }
        }
      }
      double out;
      if (mode == LS_DEMAP_MAXLOG) {
        out = mx1 - mx0;
      } else {
        double s1 = 0.0, s0 = 0.0;
        for (int p = 0; p < P; ++p) {
          if ((p >> sh) & 1) {
            if (p != a1) s1 += exp(lg[p] - mx1);
          } else {
            if (p != a0) s0 += exp(lg[p] - mx0);
          }
        }
        out = (mx1 + log1p(s1)) - (mx0 + log1p(s0));
      }
      if (llr32) llr32[s * m + j] = (float)out;
      if (llr64) llr64[s * m + j] = out;
    }
  }
}

// Gray-QAM fast path: the points are a product of two Gray
// PAM axes (even label bits -> I, odd -> Q, mapping.py:33-48), so the
// Q-axis factor cancels in every I-bit LLR and vice versa:
//   LLR(b) = LSE_{l: bit=1} -(y_ax - a_l)^2/no - LSE_{l: bit=0} (...)
// over the 2^(m/2) levels of b's own axis.  Same scipy LSE structure (max +
// log1p of the others), f64; agrees with the 2^m-point formula to ~1e-12.
struct QamAxes {
  double amp[16];   // level amplitudes (unit-energy normalised)
  int lab[16];      // axis label of each level, MSB first
};

// e^x for x <= 0 (the demapper's exp(logit - max)): x = k ln2 + r, |r| <=
// ln2/2, degree-13 Taylor for e^r (truncation < 2e-16 relative), times 2^k.
// Below -708 the reference's value is subnormal or zero, far under the f64
// resolution of the LLR it enters (log1p(t) ~ t added to a max term), so 0.
// coefficients in the constant bank: DFMA reads them as operands (as
// constexpr locals every use costs two UMOVs)
__constant__ double dm_exp_c[14] = {1.0, 1.0, 0.5, 0.16666666666666666, 0.041666666666666664, 0.008333333333333333, 0.001388888888888889, 0.0001984126984126984, 2.48015873015873e-05, 2.7557319223985893e-06, 2.755731922398589e-07, 2.505210838544172e-08, 2.08767569878681e-09, 1.6059043836821613e-10};
__constant__ double dm_atanh_c[16] = {1.0, 0.3333333333333333, 0.2, 0.14285714285714285, 0.1111111111111111, 0.09090909090909091, 0.07692307692307693, 0.06666666666666667, 0.058823529411764705, 0.05263157894736842, 0.047619047619047616, 0.043478260869565216, 0.04, 0.037037037037037035, 0.034482758620689655, 0.03225806451612903};

__device__ __forceinline__ double dm_exp_neg(double x) {
  if (x < -708.0) return 0.0;
  const double kd = rint(x * 1.4426950408889634);
  const double r = fma(kd, -1.9082149292705877e-10, fma(kd, -6.93147180369123816490e-01, x));
  double p = dm_exp_c[13];
#pragma unroll
  for (int n = 12; n >= 0; --n) p = fma(p, r, dm_exp_c[n]);
  return p * __hiloint2double(((int)kd + 1023) << 20, 0);
}

// log1p(t) for 0 <= t <= 1 (the log-sum-exp tail of a 2-level set):
// 2 atanh(z), z = t / (2 + t) <= 1/3, atanh(z)/z as its Taylor series in
// w = z^2 <= 1/9 to degree 15 (truncation < 5e-17); larger t (64/256-QAM sets
// of 4 or more levels) take the library log1p.
__device__ __forceinline__ double dm_log1p(double t) {
  if (t > 1.0) return log1p(t);
  const double z = t / (2.0 + t), w = z * z;
  double p = dm_atanh_c[15];
#pragma unroll
  for (int k = 14; k >= 0; --k) p = fma(p, w, dm_atanh_c[k]);
  return 2.0 * z * p;
}

template <int HALF, class YT>
__global__ void k_demap_qam(const YT *__restrict__ y, int64_t nsym, double no,
                            const double *__restrict__ no_vec, const double *__restrict__ prior,
                            const QamAxes A, int mode, float *__restrict__ llr32,
                            double *__restrict__ llr64) {
  constexpr int L = 1 << HALF, M = 2 * HALF;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nsym;
       s += (int64_t)gridDim.x * blockDim.x) {
    const double2 ys = ld_sym(y, s);
    const double inv = 1.0 / (no_vec ? no_vec[s] : no);
    double out[M];
#pragma unroll
    for (int ax = 0; ax < 2; ++ax) {
      const double yv = ax == 0 ? (double)ys.x : (double)ys.y;
      double lg[L];
#pragma unroll
      for (int l = 0; l < L; ++l) {
        const double d = yv - A.amp[l];
        lg[l] = -(d * d) * inv;
        if (prior) {  // the bit priors factor per axis too: bits 2t + ax of the label
          double pr = 0.0;
#pragma unroll
          for (int t = 0; t < HALF; ++t)
            if ((A.lab[l] >> (HALF - 1 - t)) & 1) pr += prior[s * M + 2 * t + ax];
          lg[l] += pr;
        }
      }
#pragma unroll
      for (int t = 0; t < HALF; ++t) {
        const int sh = HALF - 1 - t;
        double mx1 = -INFINITY, mx0 = -INFINITY;
        int a1 = -1, a0 = -1;
#pragma unroll
        for (int l = 0; l < L; ++l) {
          if ((A.lab[l] >> sh) & 1) {
            if (lg[l] > mx1) { mx1 = lg[l]; a1 = l; }
          } else {
            if (lg[l] > mx0) { mx0 = lg[l]; a0 = l; }
          }
        }
        double v;
        if (mode == LS_DEMAP_MAXLOG) {
          v = mx1 - mx0;
        } else {
          double s1 = 0.0, s0 = 0.0;
#pragma unroll
          for (int l = 0; l < L; ++l) {
            if ((A.lab[l] >> sh) & 1) {
              if (l != a1) s1 += dm_exp_neg(lg[l] - mx1);
            } else {
              if (l != a0) s0 += dm_exp_neg(lg[l] - mx0);
            }
          }
          v = (mx1 + dm_log1p(s1)) - (mx0 + dm_log1p(s0));
        }
        out[2 * t + ax] = v;  // stream bit 2t is the t-th I bit, 2t+1 the t-th Q bit
      }
    }
#pragma unroll
    for (int j = 0; j < M; ++j) {
      if (llr32) llr32[s * M + j] = (float)out[j];
      if (llr64) llr64[s * M + j] = out[j];
    }
  }
}

// Gray QAM without priors (the sweep engine's case): the same arithmetic with
// the Gray labels l ^ (l >> 1) compile-time, so every bit's two level sets,
// their maxima and the log-sum-exp tails are straight-line code
template <int HALF, int MODE, class YT>
__global__ void __launch_bounds__(256) k_demap_qam_gray(const YT *__restrict__ y, int64_t nsym, double no,
                                                        const double *__restrict__ no_vec, const QamAxes A,
                                                        float *__restrict__ llr32, double *__restrict__ llr64) {
  constexpr int L = 1 << HALF, M = 2 * HALF;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nsym;
       s += (int64_t)gridDim.x * blockDim.x) {
    const double2 ys = ld_sym(y, s);
    const double inv = 1.0 / (no_vec ? no_vec[s] : no);
    double out[M];
#pragma unroll
    for (int ax = 0; ax < 2; ++ax) {
      const double yv = ax == 0 ? (double)ys.x : (double)ys.y;
      double lg[L];
#pragma unroll
      for (int l = 0; l < L; ++l) {
        const double d = yv - A.amp[l];
        lg[l] = -(d * d) * inv;
      }
#pragma unroll
      for (int t = 0; t < HALF; ++t) {
        double lse[2];
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          // levels whose Gray label has bit t (MSB first) equal to b
          double mx = -INFINITY;
          int arg = 0;
#pragma unroll
          for (int l = 0; l < L; ++l) {
            if ((((l ^ (l >> 1)) >> (HALF - 1 - t)) & 1) != b) continue;
            if (lg[l] > mx) {
              mx = lg[l];
              arg = l;
            }
          }
          if (MODE == LS_DEMAP_MAXLOG) {
            lse[b] = mx;
          } else {
            double sum = 0.0;
#pragma unroll
            for (int l = 0; l < L; ++l) {
              if ((((l ^ (l >> 1)) >> (HALF - 1 - t)) & 1) != b) continue;
              sum += l == arg ? 0.0 : dm_exp_neg(lg[l] - mx);
            }
            lse[b] = mx + dm_log1p(sum);
          }
        }
        out[2 * t + ax] = lse[1] - lse[0];
      }
    }
#pragma unroll
    for (int j = 0; j < M; ++j) {
      if (llr32) llr32[s * M + j] = (float)out[j];
      if (llr64) llr64[s * M + j] = out[j];
    }
  }
}

// ------------------------------------------------------------ bit-packed encoder
// Row syndromes of the systematic part (ldpc.py:308-311, as XORs instead of
// the GEMM), the accumulate-core solve (ldpc.py:313-320), the extension rows
// (ldpc.py:327-331), then the rate-matching gather (ldpc.py:351), with 32
// circulant lanes per 32-bit word: a circulant
// with shift s maps word w of the output to the 32 input bits starting at
// bit 32w + s of a "doubled" copy of the input vector (bit j = x[j mod Z]),
// i.e. one funnel shift per (row, word, entry).  One CTA per codeword.
constexpr int kEncW = 12;            // max words per circulant vector (Z <= 384)
constexpr int kEncD = 2 * kEncW + 2;  // words of a doubled vector

__device__ __forceinline__ uint32_t bits_at(const uint32_t *a, int pos) {
  return __funnelshift_r(a[pos >> 5], a[(pos >> 5) + 1], pos & 31);
}

// 32 bits x[(off + b) mod Z], b = 0..31, of the Z-bit vector starting at bit
// `base` of the packed array a
__device__ __forceinline__ uint32_t bits_wrapped(const uint32_t *a, int base, int Z, int off) {
  int o = off % Z, filled = 0;
  uint32_t out = 0;
  while (filled < 32) {
    const int take = min(32 - filled, Z - o);
    uint32_t v = bits_at(a, base + o);
    if (take < 32) v &= (1u << take) - 1u;
    out |= v << filled;
    filled += take;
    o = 0;
  }
  return out;
}

template <class G>
__global__ void __launch_bounds__(128) k_encode_packed(QcParams P, const uint8_t *__restrict__ bits,
                                                       uint8_t *__restrict__ tx, uint8_t *__restrict__ full) {
  constexpr int KB = G::KB, MB = G::MB;
  __shared__ uint32_t flat[(G::NB * 384) / 32 + 2];  // systematic bits, then the whole codeword
  __shared__ uint32_t xd[KB][kEncD];               // doubled systematic columns
  __shared__ uint32_t syn[MB][kEncW];              // syndromes, then extension parities
  __shared__ uint32_t core[4][kEncW + 1];
  __shared__ uint32_t cored[4][kEncD];
  __shared__ uint32_t tmpd[kEncD];
  const int Z = P.z, W = (Z + 31) >> 5, D = 2 * W + 2, t = threadIdx.x, NT = blockDim.x;
  const uint32_t lastmask = (Z & 31) ? ((1u << (Z & 31)) - 1u) : 0xFFFFFFFFu;
  const int64_t b = blockIdx.x;
  const uint8_t *in = bits + b * (int64_t)P.k;
  const int nflat = (P.k_full + 31) >> 5;
  // 1. pack the payload (fillers are zero)
  for (int f = t; f < nflat + 2; f += NT) {
    uint32_t w = 0;
    const int j0 = f << 5;
    if (j0 + 32 <= P.k && ((reinterpret_cast<uintptr_t>(in + j0) & 15) == 0)) {
      const uint4 a = *reinterpret_cast<const uint4 *>(in + j0);
      const uint4 c = *reinterpret_cast<const uint4 *>(in + j0 + 16);
      const uint32_t q[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t v = q[k] & 0x01010101u;  // one bit per byte
        w |= ((v & 1u) | ((v >> 7) & 2u) | ((v >> 14) & 4u) | ((v >> 21) & 8u)) << (4 * k);
      }
    } else {
      for (int e = 0; e < 32; ++e) {
        const int j = j0 + e;
        if (j < P.k) w |= (uint32_t)(in[j] & 1) << e;
      }
    }
    flat[f] = w;
  }
  __syncthreads();
  // 2. doubled systematic columns
  for (int x = t; x < KB * D; x += NT) {
    const int c = x / D, q = x - c * D;
    xd[c][q] = bits_wrapped(flat, c * Z, Z, 32 * q);
  }
  __syncthreads();
  // 3. syndromes of the systematic part (ldpc.py:308-311)
  for (int x = t; x < MB * W; x += NT) {
    const int r = x / W, w = x - r * W;
    uint32_t acc = 0;
    for (int e = G::d_row_start(r); e < G::d_row_start(r + 1); ++e) {
      const int c = G::d_col(e);
      if (c < KB) acc ^= bits_at(xd[c], 32 * w + P.s[e]);
    }
    syn[r][w] = (w == W - 1) ? (acc & lastmask) : acc;
  }
  __syncthreads();
  // 4. accumulate-core solve (ldpc.py:313-320): p1 = roll(ssum, 1)
  if (t < kEncW) {
    uint32_t ss = 0;
    if (t < W) ss = syn[0][t] ^ syn[1][t] ^ syn[2][t] ^ syn[3][t];
    core[0][t] = ss;  // ssum staged in core[0]
  }
  __syncthreads();
  for (int q = t; q < D; q += NT) tmpd[q] = bits_wrapped(core[0], 0, Z, 32 * q);
  __syncthreads();
  if (t < W) {
    const uint32_t m = (t == W - 1) ? lastmask : 0xFFFFFFFFu;
    const uint32_t ss = core[0][t];
    const uint32_t p1 = bits_at(tmpd, 32 * t + Z - 1) & m;
    const uint32_t p2 = syn[0][t] ^ ss, p3 = syn[1][t] ^ p1 ^ p2, p4 = syn[2][t] ^ p3;
    core[0][t] = p1;
    core[1][t] = p2;
    core[2][t] = p3;
    core[3][t] = p4;
  }
  __syncthreads();
  for (int x = t; x < 4 * D; x += NT) {
    const int cc = x / D, q = x - cc * D;
    cored[cc][q] = bits_wrapped(core[cc], 0, Z, 32 * q);
  }
  __syncthreads();
  // 5. extension rows (ldpc.py:327-331), in place in syn[r >= 4]
  for (int x = t; x < (MB - 4) * W; x += NT) {
    const int r = 4 + x / W, w = x % W;
    uint32_t acc = syn[r][w];
    for (int e = G::d_row_start(r); e < G::d_row_start(r + 1); ++e) {
      const int c = G::d_col(e);
      if (c >= KB && c < KB + 4) acc ^= bits_at(cored[c - KB], 32 * w + P.s[e]);
    }
    syn[r][w] = (w == W - 1) ? (acc & lastmask) : acc;
  }
  __syncthreads();
  // 6. the mother codeword as one flat bit array (systematic bits are already
  //    in place in `flat`; append the parity columns)
  //    (each word is read and written by one thread only)
  uint32_t *cwf = flat;
  const int nwords = (P.n_full + 31) >> 5, w0 = P.k_full >> 5;
  for (int w = w0 + t; w < nwords + 1; w += NT) {
    uint32_t out = 0;
    int filled = 0;
    if (w == w0 && (P.k_full & 31)) {  // shared with the systematic tail
      filled = P.k_full & 31;
      out = flat[w] & ((1u << filled) - 1u);
    }
    while (filled < 32) {
      const int v = 32 * w + filled;
      if (v >= P.n_full) break;
      const int c = v / Z, i = v - c * Z;
      const int take = min(32 - filled, Z - i);
      const uint32_t *src = c < KB + 4 ? core[c - KB] : syn[c - KB];
      uint32_t bitsv = bits_at(src, i);
      if (take < 32) bitsv &= (1u << take) - 1u;
      out |= bitsv << filled;
      filled += take;
    }
    cwf[w] = out;
  }
  __syncthreads();
  // 7. outputs (ldpc.py:351): 16 rate-matched bits per thread, as one 16-byte store
  if (full) {
    for (int v = t; v < P.n_full; v += NT) full[b * (int64_t)P.n_full + v] = (uint8_t)(bits_at(cwf, v) & 1u);
  }
  if (tx) {
    uint8_t *o = tx + b * (int64_t)P.n;
    const bool al = ((reinterpret_cast<uintptr_t>(o) & 15) == 0);
    for (int j0 = 16 * t; j0 < P.n; j0 += 16 * NT) {
      const int v0 = mother_of(P, j0);
      if (al && j0 + 16 <= P.n && mother_of(P, j0 + 15) == v0 + 15) {
        const uint32_t b16 = bits_at(cwf, v0);
        uint32_t wv[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) wv[g] = (((b16 >> (4 * g)) & 15u) * 0x00204081u) & 0x01010101u;
        *reinterpret_cast<uint4 *>(o + j0) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
      } else {
        for (int j = j0; j < min(j0 + 16, P.n); ++j) o[j] = (uint8_t)(bits_at(cwf, mother_of(P, j)) & 1u);
      }
    }
  }
}

// ------------------------------------------------------------ derate_match
// ldpc.py:335-345: mother = +0.0, np.add.at over transmit_idx in index order,
// fillers = -40.
template <typename T>
__global__ void k_derate(QcParams P, const T *__restrict__ llr, int64_t batch, T *__restrict__ mother) {
  const int64_t total = batch * (int64_t)P.n_full;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t / P.n_full;
    const int v = (int)(t - b * P.n_full);
    T acc = (T)0;
    if (v >= P.k && v < P.k_full) {
      acc = (T)-40.0;
    } else if (v >= 2 * P.z) {
      const int pos = v < P.k ? v - 2 * P.z : P.l1 + (v - P.k_full);
      const T *row = llr + b * P.n;
      for (int j = pos; j < P.n; j += P.buflen) acc = acc + row[j];
    }
    mother[t] = acc;
  }
}

// ------------------------------------------------------------ count_errors
__global__ void k_count(const uint8_t *__restrict__ a, const uint8_t *__restrict__ b, int64_t len,
                        unsigned long long *__restrict__ counts) {
  const int64_t r = blockIdx.x;
  unsigned long long e = 0;
  for (int64_t j = threadIdx.x; j < len; j += blockDim.x) e += (a[r * len + j] != b[r * len + j]);
  __shared__ unsigned long long red[32];
  for (int o = 16; o; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = e;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    if (t) {
      atomicAdd(&counts[0], t);
      atomicAdd(&counts[1], 1ULL);
    }
  }
}

// ------------------------------------------------------------ hard_decide
// core.py:102-104: 1 iff L > 0 (ties and -0.0 decide 0), f32 or f64 input
template <typename T>
__global__ void k_hard(const T *__restrict__ llr, int64_t count, uint8_t *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = llr[i] > (T)0;
}

// ------------------------------------------------------------ EXIT mutual information
// ldpc.py:175-188: I = 1 - mean(log2(1 + exp(clip(-(2b-1) L, +-40)))), f64.
// Deterministic two-pass sum: fixed per-block partials, then one block.
constexpr int kMiBlocks = 1184, kMiThreads = 256;
__global__ void k_mi_partial(const double *__restrict__ llr, const double *__restrict__ bits, int64_t count,
                             double *__restrict__ part) {
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    double x = -(2.0 * bits[i] - 1.0) * llr[i];
    x = x < -40.0 ? -40.0 : (x > 40.0 ? 40.0 : x);
    acc += log2(1.0 + exp(x));
  }
  __shared__ double red[kMiThreads];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = kMiThreads / 2; o; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void k_mi_final(const double *__restrict__ part, int n, int64_t count, double *__restrict__ out) {
  __shared__ double red[kMiThreads];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += part[i];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = kMiThreads / 2; o; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double info = 1.0 - red[0] / (double)count;
    *out = info < 0.0 ? 0.0 : (info > 1.0 ? 1.0 : info);
  }
}

}  // namespace lsb

using namespace lsb;

extern "C" {

const char *ls_last_error(void) { return g_err.c_str(); }
int ls_version(void) { return 1; }

int ls_code_create(int bg, int z, int k, int n, int mb, int nb, int kb, const int32_t *entries,
                   int nnz, ls_code **out) {
  if (!out || !entries) return fail(LS_EINVAL, "ls_code_create: null argument");
  if (bg != 1 && bg != 2) return fail(LS_EINVAL, "unknown base graph " + std::to_string(bg));
  if (k < 1 || n <= k)
    return fail(LS_EINVAL, "unsupported (k=" + std::to_string(k) + ", n=" + std::to_string(n) +
                               "): need 0 < k < n");
  if (z < 2 || z > 384) return fail(LS_EINVAL, "lifting size must be in [2, 384]");
  const int wmb = bg == 1 ? BG1Tables::MB : BG2Tables::MB;
  const int wnb = bg == 1 ? BG1Tables::NB : BG2Tables::NB;
  const int wkb = bg == 1 ? BG1Tables::KB : BG2Tables::KB;
  const int wnnz = bg == 1 ? BG1Tables::NNZ : BG2Tables::NNZ;
  const int *wrow = bg == 1 ? BG1Tables::row : BG2Tables::row;
  const int *wcol = bg == 1 ? BG1Tables::col : BG2Tables::col;
  if (mb != wmb || nb != wnb || kb != wkb || nnz != wnnz)
    return fail(LS_EINVAL, "base graph dimensions do not match the compiled BG tables");
  if (k > kb * z) return fail(LS_EINVAL, "k=" + std::to_string(k) + " too large for Z");
  ls_code *c = new ls_code();
  QcParams &P = c->p;
  P.bg = bg; P.z = z; P.k = k; P.n = n; P.mb = mb; P.nb = nb; P.kb = kb; P.nnz = nnz;
  P.k_full = kb * z;
  P.n_full = nb * z;
  P.m_full = mb * z;
  P.l1 = std::max(0, k - 2 * z);
  P.buflen = P.l1 + (P.n_full - P.k_full);
  for (int e = 0; e < nnz; ++e) {
    const int r = entries[3 * e], col = entries[3 * e + 1], s = entries[3 * e + 2];
    if (r != wrow[e] || col != wcol[e]) {
      delete c;
      return fail(LS_EINVAL, "base graph entries do not match the compiled BG structure");
    }
    c->entries[3 * e] = r;
    c->entries[3 * e + 1] = col;
    c->entries[3 * e + 2] = s;
    P.s[e] = (uint16_t)(((s % z) + z) % z);
  }
  const int *wshift = bg == 1 ? BG1Tables::shift : BG2Tables::shift;
  c->std_shifts = 1;
  for (int e = 0; e < nnz; ++e) c->std_shifts &= (entries[3 * e + 2] == wshift[e]);
  *out = c;
  return LS_OK;
}

int ls_code_destroy(ls_code *code) {
  delete code;
  return LS_OK;
}

int ls_code_transmit_idx(const ls_code *code, int32_t *host_out) {
  if (!code || !host_out) return fail(LS_EINVAL, "ls_code_transmit_idx: null argument");
  for (int j = 0; j < code->p.n; ++j) host_out[j] = mother_of(code->p, j);
  return LS_OK;
}

int ls_binary_source_at(uint64_t seed, uint64_t stream_id, int64_t offset, int64_t count, uint8_t *bits,
                        void *stream) {
  if (count < 0 || offset < 0 || (!bits && count)) return fail(LS_EINVAL, "binary_source: bad arguments");
  if (offset % 32) return fail(LS_EINVAL, "binary_source: offset must be a multiple of 32 bits");
  if (!count) return LS_OK;
  const int64_t nblk = (count + 31) / 32;
  k_binary_source<<<grid_for(nblk, 256), 256, 0, as_stream(stream)>>>(seed, stream_id, offset / 32, count, bits);
  LS_CHECK_LAUNCH("ls_binary_source");
  return LS_OK;
}

int ls_binary_source(uint64_t seed, uint64_t stream_id, int64_t count, uint8_t *bits, void *stream) {
  return ls_binary_source_at(seed, stream_id, 0, count, bits, stream);
}

int ls_map_bits(const uint8_t *bits, int64_t nsym, int m, const float *points, float *x, void *stream) {
  if (m < 1 || m > 12) return fail(LS_EINVAL, "num_bits_per_symbol must be in [1, 12]");
  if (!nsym) return LS_OK;
  k_map_bits<<<grid_for(nsym, 256), 256, 0, as_stream(stream)>>>(
      bits, nsym, m, reinterpret_cast<const float2 *>(points), reinterpret_cast<float2 *>(x));
  LS_CHECK_LAUNCH("ls_map_bits");
  return LS_OK;
}

int ls_map_bits64(const uint8_t *bits, int64_t nsym, int m, const double *points64, double *x, void *stream) {
  if (m < 1 || m > 12) return fail(LS_EINVAL, "num_bits_per_symbol must be in [1, 12]");
  if (!nsym) return LS_OK;
  k_map_bits64<<<grid_for(nsym, 256), 256, 0, as_stream(stream)>>>(
      bits, nsym, m, reinterpret_cast<const double2 *>(points64), reinterpret_cast<double2 *>(x));
  LS_CHECK_LAUNCH("ls_map_bits64");
  return LS_OK;
}

int ls_awgn_at(const float *x, int64_t offset, int64_t count, double no, uint64_t seed, uint64_t stream_id,
               float *y, void *stream) {
  if (no < 0) return fail(LS_EINVAL, "noise variance must be >= 0, got " + std::to_string(no));
  if (offset < 0 || (offset & 1)) return fail(LS_EINVAL, "awgn: offset must be even and >= 0");
  if (!count) return LS_OK;
  if (no == 0) {
    cudaError_t e = cudaMemcpyAsync(y, x, (size_t)count * 8, cudaMemcpyDeviceToDevice, as_stream(stream));
    return e == cudaSuccess ? LS_OK : cuda_status(e, "ls_awgn");
  }
  k_awgn<<<grid_for((count + 1) / 2, 256), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const float2 *>(x), count, (float)sqrt(no / 2.0), seed, stream_id, offset / 2,
      reinterpret_cast<float2 *>(y));
  LS_CHECK_LAUNCH("ls_awgn");
  return LS_OK;
}

int ls_awgn(const float *x, int64_t count, double no, uint64_t seed, uint64_t stream_id, float *y,
            void *stream) {
  return ls_awgn_at(x, 0, count, no, seed, stream_id, y, stream);
}

}  // extern "C"

template <class YT>
static int demap_any(const YT *yy, int64_t nsym, double no, const double *no_vec, const double *prior,
                     const double *points64, int m, int mode, float *llr32, double *llr64, void *stream) {
  if (!no_vec && !(no > 0)) return fail(LS_EINVAL, "demap: noise variance must be > 0");
  if (m < 1 || m > 8) return fail(LS_EINVAL, "demap: num_bits_per_symbol must be in [1, 8]");
  if (mode != LS_DEMAP_APP && mode != LS_DEMAP_MAXLOG) return fail(LS_EINVAL, "demap: unknown mode");
  if (!nsym) return LS_OK;
  const double2 *pp = reinterpret_cast<const double2 *>(points64);
  cudaStream_t s = as_stream(stream);
  if (m <= 4)
    k_demap<16><<<grid_for(nsym, 128), 128, 0, s>>>(yy, nsym, no, no_vec, prior, pp, m, mode, llr32, llr64);
  else if (m <= 6)
    k_demap<64><<<grid_for(nsym, 128), 128, 0, s>>>(yy, nsym, no, no_vec, prior, pp, m, mode, llr32, llr64);
  else
    k_demap<256><<<grid_for(nsym, 64), 64, 0, s>>>(yy, nsym, no, no_vec, prior, pp, m, mode, llr32, llr64);
  LS_CHECK_LAUNCH("ls_demap");
  return LS_OK;
}

extern "C" {

int ls_demap(const float *y, int64_t nsym, double no, const double *no_vec, const double *prior,
             const double *points64, int m, int mode, float *llr32, double *llr64, void *stream) {
  return demap_any(reinterpret_cast<const float2 *>(y), nsym, no, no_vec, prior, points64, m, mode, llr32, llr64,
                   stream);
}

int ls_demap64(const double *y, int64_t nsym, double no, const double *no_vec, const double *prior,
               const double *points64, int m, int mode, float *llr32, double *llr64, void *stream) {
  return demap_any(reinterpret_cast<const double2 *>(y), nsym, no, no_vec, prior, points64, m, mode, llr32, llr64,
                   stream);
}

}  // extern "C"

template <class YT>
static int demap_qam_any(const YT *yy, int64_t nsym, double no, const double *no_vec, const double *prior,
                         const double *amp, const int32_t *lab, int m, int mode, float *llr32, double *llr64,
                         void *stream) {
  if (!no_vec && !(no > 0)) return fail(LS_EINVAL, "demap: noise variance must be > 0");
  if (m < 2 || m > 8 || (m % 2)) return fail(LS_EINVAL, "demap_qam: bits per symbol must be 2, 4, 6 or 8");
  if (mode != LS_DEMAP_APP && mode != LS_DEMAP_MAXLOG) return fail(LS_EINVAL, "demap: unknown mode");
  if (!amp || !lab) return fail(LS_EINVAL, "demap_qam: null level table");
  if (!nsym) return LS_OK;
  QamAxes A;
  const int L = 1 << (m / 2);
  for (int l = 0; l < 16; ++l) {
    A.amp[l] = l < L ? amp[l] : 0.0;
    A.lab[l] = l < L ? lab[l] : 0;
  }
  cudaStream_t s = as_stream(stream);
  const unsigned g = grid_for(nsym, 256);
  bool gray = !prior && (m == 4 || m == 6);
  for (int l = 0; l < L; ++l) gray = gray && lab[l] == (l ^ (l >> 1));
  if (gray) {
    if (m == 4) {
      if (mode == LS_DEMAP_APP)
        k_demap_qam_gray<2, LS_DEMAP_APP><<<g, 256, 0, s>>>(yy, nsym, no, no_vec, A, llr32, llr64);
      else
        k_demap_qam_gray<2, LS_DEMAP_MAXLOG><<<g, 256, 0, s>>>(yy, nsym, no, no_vec, A, llr32, llr64);
    } else {
      if (mode == LS_DEMAP_APP)
        k_demap_qam_gray<3, LS_DEMAP_APP><<<g, 256, 0, s>>>(yy, nsym, no, no_vec, A, llr32, llr64);
      else
        k_demap_qam_gray<3, LS_DEMAP_MAXLOG><<<g, 256, 0, s>>>(yy, nsym, no, no_vec, A, llr32, llr64);
    }
    LS_CHECK_LAUNCH("ls_demap_qam");
    return LS_OK;
  }
  switch (m) {
    case 2: k_demap_qam<1><<<g, 256, 0, s>>>(yy, nsym, no, no_vec, prior, A, mode, llr32, llr64); break;
    case 4: k_demap_qam<2><<<g, 256, 0, s>>>(yy, nsym, no, no_vec, prior, A, mode, llr32, llr64); break;
    case 6: k_demap_qam<3><<<g, 256, 0, s>>>(yy, nsym, no, no_vec, prior, A, mode, llr32, llr64); break;
    default: k_demap_qam<4><<<g, 256, 0, s>>>(yy, nsym, no, no_vec, prior, A, mode, llr32, llr64); break;
  }
  LS_CHECK_LAUNCH("ls_demap_qam");
  return LS_OK;
}

extern "C" {

int ls_demap_qam(const float *y, int64_t nsym, double no, const double *no_vec, const double *prior,
                 const double *amp, const int32_t *lab, int m, int mode, float *llr32, double *llr64,
                 void *stream) {
  return demap_qam_any(reinterpret_cast<const float2 *>(y), nsym, no, no_vec, prior, amp, lab, m, mode, llr32,
                       llr64, stream);
}

int ls_demap_qam64(const double *y, int64_t nsym, double no, const double *no_vec, const double *prior,
                   const double *amp, const int32_t *lab, int m, int mode, float *llr32, double *llr64,
                   void *stream) {
  return demap_qam_any(reinterpret_cast<const double2 *>(y), nsym, no, no_vec, prior, amp, lab, m, mode, llr32,
                       llr64, stream);
}

int ls_modem_qam(const uint8_t *bits, int64_t nsym, int m, const float *points, const double *amp,
                 const int32_t *lab, double no, uint64_t seed, uint64_t stream_id, int mode, float *llr,
                 void *stream) {
  return ls_modem_qam_at(bits, 0, nsym, m, points, amp, lab, no, seed, stream_id, mode, llr, stream);
}

int ls_modem_qam_at(const uint8_t *bits, int64_t offset, int64_t nsym, int m, const float *points,
                    const double *amp, const int32_t *lab, double no, uint64_t seed, uint64_t stream_id,
                    int mode, float *llr, void *stream) {
  if (!(no > 0)) return fail(LS_EINVAL, "demap: noise variance must be > 0");
  if (offset < 0 || (offset & 1)) return fail(LS_EINVAL, "modem_qam: offset must be even and >= 0");
  if (m < 2 || m > 8 || (m % 2)) return fail(LS_EINVAL, "modem_qam: bits per symbol must be 2, 4, 6 or 8");
  if (mode != LS_DEMAP_APP && mode != LS_DEMAP_MAXLOG) return fail(LS_EINVAL, "demap: unknown mode");
  if (!nsym) return LS_OK;
  QamAxesF A;
  const int L = 1 << (m / 2);
  for (int l = 0; l < 16; ++l) {
    A.amp[l] = l < L ? (float)amp[l] : 0.0f;
    A.lab[l] = l < L ? lab[l] : 0;
    if (l < L && lab[l] != (l ^ (l >> 1)))
      return fail(LS_EINVAL, "modem_qam: levels must carry the Gray labels l ^ (l >> 1)");
  }
  const float2 *pp = reinterpret_cast<const float2 *>(points);
  const float sigma = (float)sqrt(no / 2.0), inv = (float)(1.0 / no);
  const int ml = mode == LS_DEMAP_MAXLOG;
  cudaStream_t s = as_stream(stream);
  const unsigned g = grid_for((nsym + 1) / 2, 256);
  const int64_t q0 = offset / 2;
  const bool vec = ((uintptr_t)bits % 4 == 0) && ((uintptr_t)llr % 16 == 0);
#define LSB_MODEM(H)                                                                                           \
  (vec ? k_modem_qam<H, true><<<g, 256, 0, s>>>(bits, nsym, pp, sigma, inv, seed, stream_id, q0, A, ml, llr) \
       : k_modem_qam<H, false><<<g, 256, 0, s>>>(bits, nsym, pp, sigma, inv, seed, stream_id, q0, A, ml, llr))
  switch (m) {
    case 2: LSB_MODEM(1); break;
    case 4: LSB_MODEM(2); break;
    case 6: LSB_MODEM(3); break;
    default: LSB_MODEM(4); break;
  }
#undef LSB_MODEM
  LS_CHECK_LAUNCH("ls_modem_qam");
  return LS_OK;
}

int ls_encode(const ls_code *code, const uint8_t *bits, int64_t batch, uint8_t *tx, uint8_t *full,
              void *stream) {
  if (!code) return fail(LS_EINVAL, "ls_encode: null code");
  if (!batch) return LS_OK;
  const QcParams &P = code->p;
  cudaStream_t s = as_stream(stream);
  if (P.bg == 1)
    k_encode_packed<BG1Tables><<<(unsigned)batch, 128, 0, s>>>(P, bits, tx, full);
  else
    k_encode_packed<BG2Tables><<<(unsigned)batch, 128, 0, s>>>(P, bits, tx, full);
  LS_CHECK_LAUNCH("ls_encode");
  return LS_OK;
}

int ls_derate(const ls_code *code, const void *llr, int is_f64, int64_t batch, void *mother, void *stream) {
  if (!code) return fail(LS_EINVAL, "ls_derate: null code");
  if (!batch) return LS_OK;
  const int64_t total = batch * code->p.n_full;
  cudaStream_t s = as_stream(stream);
  if (is_f64)
    k_derate<double><<<grid_for(total, 256), 256, 0, s>>>(code->p, (const double *)llr, batch, (double *)mother);
  else
    k_derate<float><<<grid_for(total, 256), 256, 0, s>>>(code->p, (const float *)llr, batch, (float *)mother);
  LS_CHECK_LAUNCH("ls_derate");
  return LS_OK;
}

int ls_hard_decide(const void *llr, int is_f64, int64_t count, uint8_t *out, void *stream) {
  if (count < 0 || (count && (!llr || !out))) return fail(LS_EINVAL, "hard_decide: bad arguments");
  if (!count) return LS_OK;
  cudaStream_t s = as_stream(stream);
  if (is_f64)
    k_hard<double><<<grid_for(count, 256), 256, 0, s>>>((const double *)llr, count, out);
  else
    k_hard<float><<<grid_for(count, 256), 256, 0, s>>>((const float *)llr, count, out);
  LS_CHECK_LAUNCH("ls_hard_decide");
  return LS_OK;
}

int ls_exit_mutual_information(const double *llr, const double *bits, int64_t count, double *out, void *stream) {
  if (count <= 0) return fail(LS_EINVAL, "exit_mutual_information: empty input");
  if (!llr || !bits || !out) return fail(LS_EINVAL, "exit_mutual_information: null argument");
  cudaStream_t s = as_stream(stream);
  double *part = nullptr;
  cudaError_t e = cudaMallocAsync((void **)&part, sizeof(double) * kMiBlocks, s);
  if (e != cudaSuccess) return cuda_status(e, "exit_mutual_information(workspace)");
  k_mi_partial<<<kMiBlocks, kMiThreads, 0, s>>>(llr, bits, count, part);
  k_mi_final<<<1, kMiThreads, 0, s>>>(part, kMiBlocks, count, out);
  e = cudaGetLastError();
  cudaFreeAsync(part, s);
  return e == cudaSuccess ? LS_OK : cuda_status(e, "exit_mutual_information");
}

int ls_count_errors(const uint8_t *b, const uint8_t *b_hat, int64_t batch, int64_t len,
                    unsigned long long *counts, void *stream) {
  if (!batch || !len) return LS_OK;
  k_count<<<(unsigned)batch, 256, 0, as_stream(stream)>>>(b, b_hat, len, counts);
  LS_CHECK_LAUNCH("ls_count_errors");
  return LS_OK;
}

}  // extern "C"
