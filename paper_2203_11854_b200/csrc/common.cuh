// Shared device/host helpers for the linksim_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/linksim_b200.h"
#include "bg_tables.h"

namespace lsb {

// ---------------------------------------------------------------- errors
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);
int cuda_status(cudaError_t e, const char *where);

#define LS_CHECK_LAUNCH(where)                                      \
  do {                                                              \
    cudaError_t _e = cudaGetLastError();                            \
    if (_e != cudaSuccess) return ::lsb::cuda_status(_e, where);    \
  } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// keep the stream-ordered allocator's memory between calls (workspaces of the
// exact decoder and of the numpy-normal replica are GB-sized)
void retain_pool_memory();

inline unsigned grid_for(int64_t n, int block, int64_t cap = 148LL * 64) {
  int64_t g = (n + block - 1) / block;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (unsigned)g;
}

// ---------------------------------------------------------------- code handle
constexpr int kMaxNnz = 336;

// Everything a QC kernel needs about one lifted code + rate matching,
// passed BY VALUE as a kernel parameter (it lands in the constant bank, so
// the per-entry shifts are free uniform operands).
struct QcParams {
  int bg, z, k, n;
  int mb, nb, kb, nnz;
  int k_full, n_full, m_full;
  int l1;      // length of the first buffer segment [2Z, k)
  int buflen;  // circular-buffer length (ldpc.py:252-255)
  uint16_t s[kMaxNnz];  // shift mod z per base entry, (row, col) order
};

// Flush-to-zero approximate MUFU forms: one SFU instruction each, without
// the denormal fix-ups the default intrinsics carry (for operands known to be
// normal floats).
__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2_ftz(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_ftz(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sqrt_ftz(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sin_ftz(float x) {
  float y;
  asm("sin.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float cos_ftz(float x) {
  float y;
  asm("cos.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
constexpr float kLn2 = 0.693147180559945309f, kLog2e = 1.442695040888963407f;

}  // namespace lsb

struct ls_code {
  lsb::QcParams p;
  int32_t entries[3 * lsb::kMaxNnz];
  int std_shifts;  // shifts equal the compiled base-graph tables (specialised kernels usable)
};

struct ls_graph {
  int64_t n, m, E;
  int max_cdeg, max_vdeg;
  int32_t *cptr;   // [m+1] device
  int32_t *cvar;   // [E]   device
  int32_t *vptr;   // [n+1] device
  int32_t *vedge;  // [E]   device: edges of each VN, ascending check order
};

namespace lsb {

// rate-matched position -> mother index (closed form of transmit_idx,
// ldpc.py:249-256): buffer = [2Z, k) U [k_full, n_full)
__host__ __device__ inline int mother_of(const QcParams &P, int j) {
  int p = j % P.buflen;
  return p < P.l1 ? 2 * P.z + p : P.k_full + (p - P.l1);
}

// ---------------------------------------------------------------- Philox
// numpy's Philox4x64-10, keyed (k0, k1) = (stream_id, seed).
__device__ __forceinline__ void philox4x64_10(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3,
                                              uint64_t k0, uint64_t k1, uint64_t out[4]) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B97F4A7C15ULL;
      k1 += 0xBB67AE8584CAA73BULL;
    }
    uint64_t lo0 = 0xD2E7470EE14C6C93ULL * c0, hi0 = __umul64hi(0xD2E7470EE14C6C93ULL, c0);
    uint64_t lo1 = 0xCA5A826395121157ULL * c2, hi1 = __umul64hi(0xCA5A826395121157ULL, c2);
    uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

// Philox4x32-10 (Salmon et al. 2011) for the fast-mode noise stream.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  return c;
}

}  // namespace lsb
