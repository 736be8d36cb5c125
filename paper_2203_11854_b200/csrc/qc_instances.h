// Specialised fast-decoder instances compiled in: (base graph, Z, processed
// rows, threads per lane, kind).  Each becomes build/gen/qc_<...>.cu.
// fp16x2 min-sum codes matching none of them use a runtime-geometry instance
// (LSB_QC_RT_INSTANCES below); fp32 ones the runtime-Z kernel in bp_fast.cu;
// sum-product fast mode uses these instances or a runtime-geometry one
// (LSB_QC_SPRT_INSTANCES) when its messages fit in shared memory.
//   1,384,24 / 1,384,46 : config 2 (k=8448 n=16896), dead rows pruned / all
//   1,192,{24,45,46}    : configs 3 and 4 (k=4096, n=8192 / 12288)
//   2,26,{12,42}        : config 1 (k=256 n=512)
//   1,Z,24 / 2,Z,22 for Z in 32..384 : config 5 decoder-only sweep (BG1 rate
//                         1/2 and BG2 rate 1/3 lifted at any Z, fp16x2)
// kind f32: k_qc_fast2 (bp_fast_qc.cuh); h2: k_qc_fast_h2 (bp_fast_h2.cuh);
// sp: k_qc_sp, sum-product (bp_fast_sp.cuh); sp32: k_qc_sp32, sum-product with
// f32 messages and the product-domain check update (accuracy option; at
// Z = 384 the messages live in an L2 slice per CTA)
#pragma once
#define LSB_QC_INSTANCES(X) \
  X(1, 384, 24, 2, f32)     \
  X(1, 384, 46, 2, f32)     \
  X(1, 192, 24, 4, f32)     \
  X(1, 192, 45, 2, f32)     \
  X(1, 192, 46, 2, f32)     \
  X(2, 26, 12, 1, f32)      \
  X(2, 26, 42, 1, f32)      \
  X(1, 384, 24, 2, h2)      \
  X(1, 384, 46, 2, h2)      \
  X(1, 192, 24, 4, h2)      \
  X(1, 192, 45, 2, h2)      \
  X(1, 192, 46, 2, h2)      \
  X(2, 26, 12, 1, h2)       \
  X(2, 26, 42, 1, h2)       \
  X(1, 32, 24, 4, h2)       \
  X(1, 64, 24, 4, h2)       \
  X(1, 128, 24, 4, h2)      \
  X(1, 256, 24, 2, h2)      \
  X(2, 32, 22, 4, h2)       \
  X(2, 64, 22, 4, h2)       \
  X(2, 128, 22, 4, h2)      \
  X(2, 192, 22, 4, h2)      \
  X(2, 256, 22, 2, h2)      \
  X(2, 384, 22, 2, h2)      \
  X(1, 384, 24, 2, sp)      \
  X(1, 192, 24, 2, sp)      \
  X(1, 192, 45, 2, sp)      \
  X(1, 192, 46, 2, sp)      \
  X(2, 26, 12, 1, sp)       \
  X(2, 26, 42, 1, sp)       \
  X(1, 384, 24, 1, sp32)    \
  X(1, 192, 24, 2, sp32)    \
  X(2, 26, 12, 1, sp32)     \
  X(2, 26, 42, 1, sp32)

// Runtime-geometry fp16x2 instances (base graph, row bound RB, threads per
// lane): any Z <= 384 (<= 192 with 4 threads per lane) and any processed-row
// count R <= RB.  The dispatcher picks the smallest RB >= R that fits.
#define LSB_QC_RT_INSTANCES(Y) \
  Y(1, 12, 2)                  \
  Y(1, 24, 2)                  \
  Y(1, 46, 2)                  \
  Y(1, 46, 4)                  \
  Y(2, 12, 2)                  \
  Y(2, 22, 2)                  \
  Y(2, 42, 2)                  \
  Y(2, 42, 4)

// Runtime-geometry sum-product instances (base graph, row bound RB, threads
// per lane); per-edge fp16 messages must fit in shared memory.
#define LSB_QC_SPRT_INSTANCES(W) \
  W(1, 24, 2)                    \
  W(1, 46, 2)                    \
  W(2, 22, 2)                    \
  W(2, 42, 2)

// On-chip EXACT-mode decoders (bp_qc_exact.cuh): base graph, Z, thread
// groups per lane.  Bit-identical min-sum / scaled-min-sum on the whole
// mother graph; codes without an instance use the HBM-streaming CSR decoder
// (bp_exact.cu).
//   1,384 : config 2        1,192 : configs 3 and 4       2,26 : config 1
//   1,64 / 2,64 / 2,384 : config 5's decoder-only geometries
#define LSB_QCX_INSTANCES(V) \
  V(1, 384, 2)               \
  V(1, 192, 2)               \
  V(1, 64, 2)                \
  V(2, 384, 2)               \
  V(2, 64, 2)                \
  V(2, 26, 2)
