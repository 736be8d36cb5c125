/*
 * linksim_b200 -- C ABI of the B200 (sm_100a) coded-link hot path.
 *
 * Drop-in boundary for the reference's module-level block functions
 * (linksim 0.1.0, /root/reference/pkg/src/linksim).  The reference is pure
 * Python/numpy; each entry point below replaces the numpy body of one
 * reference function (cited per function) while the Python signatures are
 * mirrored 1:1 by paper_2203_11854_b200/*.py, which binds this library with
 * ctypes (see INTEGRATION.md for the stub a linksim maintainer would add).
 *
 * Conventions
 *   - Every array pointer is a DEVICE pointer owned by the caller, row-major
 *     with the Monte-Carlo batch on the leading axis (core.py:4-7).
 *     Bits are uint8 in {0,1}; complex values are interleaved (re, im).
 *   - `stream` is a cudaStream_t passed as void*; all work is enqueued on it
 *     and the call returns without synchronising (except where noted).
 *   - Return value is LS_OK (0) or an LS_E* status; ls_last_error() returns a
 *     thread-local message.  Invalid arguments are reported with the same
 *     wording as the reference's ValueErrors (ldpc.py:108-114, 228-231;
 *     channel.py:36-37; mapping.py:113-114).
 *   - Handles are immutable after creation and may be shared by threads
 *     (run_sweep drives run_batch from a thread pool, sweep.py:425-449).
 */
#ifndef LINKSIM_B200_H
#define LINKSIM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LS_OK 0
#define LS_EINVAL 1 /* bad argument (Python side raises ValueError) */
#define LS_ECUDA 2  /* CUDA runtime error */
#define LS_ENOMEM 3

/* BP variants, ldpc.py:23 BP_VARIANTS order */
#define LS_SUM_PRODUCT 0
#define LS_MIN_SUM 1
#define LS_SCALED_MIN_SUM 2

/* demapper modes, mapping.py:146-158 */
#define LS_DEMAP_APP 0
#define LS_DEMAP_MAXLOG 1

typedef struct ls_code ls_code;   /* lifted QC code + rate matching (LdpcCode5G) */
typedef struct ls_graph ls_graph; /* generic check-major CSR Tanner graph     */

const char *ls_last_error(void);
int ls_version(void);

/* ---- code handles ---------------------------------------------------- */
/* LdpcCode5G(k, n) (ldpc.py:214-272): base graph `bg` with m_b x n_b blocks,
 * k_b systematic columns, `nnz` (row, col, shift) entries sorted by
 * (row, col) (ldpc.py:191-202), lifting size z.  Shifts are reduced mod z
 * here (ldpc.py:263, 288). */
int ls_code_create(int bg, int z, int k, int n, int mb, int nb, int kb,
                   const int32_t *entries, int nnz, ls_code **out);
int ls_code_destroy(ls_code *code);
/* transmit_idx of the code (ldpc.py:252-256) into a host int32[n] buffer. */
int ls_code_transmit_idx(const ls_code *code, int32_t *host_out);

/* ParityCheckMatrix as CSR (alist.py:25-58): check c owns edges
 * [cptr[c], cptr[c+1]) whose variables cvar[] ascend (host pointers). */
int ls_graph_create(int64_t n, int64_t m, const int64_t *cptr, const int64_t *cvar,
                    ls_graph **out);
/* The lifted mother-code graph of a QC code (LdpcCode5G.pcm, ldpc.py:278-296). */
int ls_graph_from_code(const ls_code *code, ls_graph **out);
int ls_graph_destroy(ls_graph *g);

/* ---- sources and channel --------------------------------------------- */
/* binary_source(shape, RngStream(seed, stream_id)) (core.py:47-54): bit-exact
 * replica of numpy's Philox4x64-10 + bounded uint8 draw, `count` bits. */
int ls_binary_source(uint64_t seed, uint64_t stream_id, int64_t count, uint8_t *bits,
                     void *stream);

/* map_bits(bits, constellation) (mapping.py:96-107): big-endian m-bit
 * groups index `points` (2^m complex64, interleaved, device).  nsym symbols. */
int ls_map_bits(const uint8_t *bits, int64_t nsym, int m, const float *points, float *x,
                void *stream);
/* The same into complex128 (precision "double", sweep.py:170, 352): points64
 * are the f64 constellation points. */
int ls_map_bits64(const uint8_t *bits, int64_t nsym, int m, const double *points64, double *x,
                  void *stream);

/* awgn(x, no, rng) (channel.py:33-40) for complex64 x: x + sqrt(no/2) * z with
 * z drawn from a counter-based Philox4x32-10 / Box-Muller stream keyed by
 * (seed, stream_id).  Statistically equivalent to the reference (fast
 * mode); ls_awgn_numpy below is the bit-exact numpy-ziggurat replica. */
int ls_awgn(const float *x, int64_t count, double no, uint64_t seed, uint64_t stream_id, float *y,
            void *stream);

/* Bit-exact replicas of the reference's numpy draws (channel.py:24-40):
 * ls_standard_normal = `count` draws of Generator.standard_normal on
 * RngStream(seed, stream_id) (numpy 2.3.5 ziggurat, f64);
 * ls_awgn_numpy = awgn(x, no, rng) for complex64 x with exactly the
 * reference's noise: real parts = normals [0, count), imaginary parts =
 * normals [count, 2*count), scaled by sqrt(no/2) in f64, cast to f32, added. */
int ls_standard_normal(uint64_t seed, uint64_t stream_id, int64_t count, double *out, void *stream);
int ls_awgn_numpy(const float *x, int64_t count, double no, uint64_t seed, uint64_t stream_id,
                  float *y, void *stream);
/* awgn for complex128 x (precision "double"): the same normals, noise kept
 * in f64 and added in f64 (channel.py:27-40 with dtype complex128). */
int ls_awgn_numpy64(const double *x, int64_t count, double no, uint64_t seed, uint64_t stream_id,
                    double *y, void *stream);

/* demap_app / demap_maxlog (mapping.py:110-158) for any 2^m points:
 * y complex64 [nsym], scalar no (>0) or per-symbol `no_vec` (nullable),
 * optional per-bit priors `prior` [nsym, m] (LLR, added to the logits of the
 * points whose bit is 1, mapping.py:123-131; nullable), f64 log-domain
 * arithmetic; llr written as f32 (`llr32`) or f64 (`llr64`), whichever is
 * non-null, m values per symbol. */
int ls_demap(const float *y, int64_t nsym, double no, const double *no_vec, const double *prior,
             const double *points64, int m, int mode, float *llr32, double *llr64, void *stream);
/* ls_demap / ls_demap_qam on complex128 symbols (precision "double"). */
int ls_demap64(const double *y, int64_t nsym, double no, const double *no_vec, const double *prior,
               const double *points64, int m, int mode, float *llr32, double *llr64, void *stream);

/* Same as ls_demap for Gray QAM (mapping.py:33-48), using the product
 * structure: each bit's LLR is a log-sum-exp over the 2^(m/2) levels of its
 * own axis (equal to the 2^m-point formula to ~1e-12).
 * amp[l] / lab[l] (host, 2^(m/2) entries): amplitude and axis label of level l. */
int ls_demap_qam(const float *y, int64_t nsym, double no, const double *no_vec,
                 const double *prior, const double *amp, const int32_t *lab, int m, int mode,
                 float *llr32, double *llr64, void *stream);
int ls_demap_qam64(const double *y, int64_t nsym, double no, const double *no_vec,
                   const double *prior, const double *amp, const int32_t *lab, int m, int mode,
                   float *llr32, double *llr64, void *stream);

/* Fused map_bits -> awgn -> demap_app|maxlog for Gray QAM (sweep.py:352-356
 * in one pass): coded bits [nsym*m] -> f32 LLRs [nsym*m].  The noisy symbols
 * equal ls_map_bits + ls_awgn with the same (seed, stream_id); the per-axis
 * log-sum-exp runs in f32.  points: 2^m complex64 (device); amp/lab as in
 * ls_demap_qam (host; lab[l] must be the Gray label l ^ (l >> 1)). */
int ls_modem_qam(const uint8_t *bits, int64_t nsym, int m, const float *points, const double *amp,
                 const int32_t *lab, double no, uint64_t seed, uint64_t stream_id, int mode,
                 float *llr, void *stream);

/* Slice variants for chunked (copy-overlapped) batches: the same streams as
 * one call over the whole array, starting at element `offset` of it
 * (binary_source: bit offset, multiple of 32; awgn / modem: complex
 * element / symbol offset, even). */
int ls_binary_source_at(uint64_t seed, uint64_t stream_id, int64_t offset, int64_t count,
                        uint8_t *bits, void *stream);
int ls_awgn_at(const float *x, int64_t offset, int64_t count, double no, uint64_t seed,
               uint64_t stream_id, float *y, void *stream);
int ls_modem_qam_at(const uint8_t *bits, int64_t offset, int64_t nsym, int m, const float *points,
                    const double *amp, const int32_t *lab, double no, uint64_t seed,
                    uint64_t stream_id, int mode, float *llr, void *stream);

/* ---- LDPC ------------------------------------------------------------ */
/* ldpc5g_encode(bits, code) (ldpc.py:298-351): bits [B,k] -> rate-matched
 * codewords tx [B,n] (nullable) and/or the mother codeword full [B,n_full]
 * (nullable, encode_full). */
int ls_encode(const ls_code *code, const uint8_t *bits, int64_t batch, uint8_t *tx,
              uint8_t *full, void *stream);

/* derate_match (ldpc.py:335-345): llr [B,n] -> mother [B,n_full], f32 or f64. */
int ls_derate(const ls_code *code, const void *llr, int is_f64, int64_t batch, void *mother,
              void *stream);

/* bp_decode(llr, pcm, num_iter, variant, scale, early_stop) (ldpc.py:86-172),
 * EXACT mode: reproduces the reference arithmetic (f64 messages, numpy
 * reduceat summation order, f32 posterior rounding for f32 input, per-row
 * early stop).  llr [B,n] f32 (is_f64=0) or f64; outputs llr_out [B,n] same
 * dtype, hard [B,n] uint8, iters_used [B] int32 (nullable). */
int ls_bp_decode(const ls_graph *g, const void *llr, int is_f64, int64_t batch, int num_iter,
                 int variant, double scale, int early_stop, void *llr_out, uint8_t *hard,
                 int32_t *iters_used, void *stream);

/* ldpc5g_decode (ldpc.py:354-365) FAST mode on the QC structure, fused with
 * derate_match, hard decision (core.py:102-104) and count_errors
 * (core.py:93-99), messages on chip.  The fp16x2 kernels run a pair of
 * codewords per CTA (persistent CTAs, one or two slots per SM); the exact /
 * fp32 full-graph kernel (LS_QC_EXACT / LS_QC_FULL32) one codeword per
 * persistent CTA at Z = 384 and 384 / Z codewords in lockstep below it.
 * llr [B,n] f32
 * rate-matched.  Outputs (all nullable): hard_k [B,k] info bits,
 * llr_out [B,n_full] f32 mother LLRs (ln p1/p0), iters_used [B],
 * counts[2] += (bit errors, block errors) against ref_bits [B,k].
 * flags: LS_QC_PRUNE skips the dead extension rows whose parity bit is never
 * transmitted (their llr_out entries are then the channel values);
 * LS_QC_GENERIC forces a runtime-geometry kernel instead of a specialised
 * one (fp32: the runtime-Z kernel; with LS_QC_FP16: the runtime-geometry
 * fp16x2 kernel, which is also what LS_QC_FP16 uses when no specialised
 * instance exists). */
#define LS_QC_PRUNE 1
#define LS_QC_GENERIC 2
#define LS_QC_FP16 4 /* packed fp16x2 kernel: two codewords per 32-bit lane */
#define LS_QC_SP 8   /* ls_qc_has_kernel only: ask for the sum-product kernel */
/* LS_QC_EXACT: the on-chip EXACT decoder (min-sum / scaled-min-sum only):
 * bit-identical llr_out, hard decisions and iteration counts to the
 * reference bp_decode on the whole mother graph (ldpc.py:86-172; never
 * pruned), f64 messages held as a compressed per-check state in shared
 * memory + L2.  With LS_QC_MOTHER the input is mother LLRs [B,n_full]
 * (bp_decode on code.pcm, no derate) and hard_k receives [B,n_full]. */
#define LS_QC_EXACT 16
#define LS_QC_MOTHER 32
/* LS_QC_FULL32: the same on-chip decoder with f32 messages (fp32 full-graph
 * fast mode: f32 v2c / min tracking / variable sums, all rows, compressed
 * state wholly in shared memory); LLRs within tolerance of exact mode.  With
 * variant sum-product it selects k_qc_sp32 (f32 messages, log-domain check
 * update, the reference's f32 first pass) where its messages fit. */
#define LS_QC_FULL32 64
int ls_qc_decode(const ls_code *code, const float *llr, int64_t batch, int num_iter, int variant,
                 double scale, int early_stop, int flags, uint8_t *hard_k, float *llr_out,
                 int32_t *iters_used, const uint8_t *ref_bits, unsigned long long *counts,
                 void *stream);
/* Number of base rows the fast decoder processes with LS_QC_PRUNE. */
int ls_qc_live_rows(const ls_code *code);
/* 1 if a compile-time specialised kernel serves this code with these flags
 * (LS_QC_PRUNE / LS_QC_FP16), else 0 (fp32 falls back to the runtime-Z kernel). */
int ls_qc_has_kernel(const ls_code *code, int flags);

/* hard_decide(llr) (core.py:102-104): out[i] = llr[i] > 0, f32 or f64. */
int ls_hard_decide(const void *llr, int is_f64, int64_t count, uint8_t *out, void *stream);

/* exit_mutual_information(llr, bits) (ldpc.py:175-188): writes
 * clip(1 - mean(log2(1 + exp(clip(-(2b-1) L, +-40)))), 0, 1) to *out
 * (device f64); bits as f64 {0, 1}.  Deterministic reduction order. */
int ls_exit_mutual_information(const double *llr, const double *bits, int64_t count, double *out,
                               void *stream);

/* count_errors(b, b_hat) (core.py:93-99): counts[2] += (bit, block) errors. */
int ls_count_errors(const uint8_t *b, const uint8_t *b_hat, int64_t batch, int64_t len,
                    unsigned long long *counts, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* LINKSIM_B200_H */
