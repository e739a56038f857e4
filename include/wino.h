/* wino.h -- C ABI of the B200 (sm_100a) hot path of arXiv 2201.10369
 * ("symmetric interpolation points for Winograd / Toom-Cook convolution").
 *
 * Citations are PAPER.md line numbers (P:n); readings of the paper are numbered
 * R1.. in DESIGN.md §2.
 *
 * Conventions (all calls):
 *  - Plain C types only.  The caller owns every buffer; the library keeps no pointer
 *    after a call returns and allocates no device memory (scratch comes from the
 *    caller's workspace).  No C++ exception crosses the ABI.
 *  - Return value: WINO_OK or a wino_status.  Argument / shape errors are detected
 *    synchronously before any device work is enqueued; wino_last_error() then holds a
 *    thread-local message.  Device faults surface at the caller's next synchronisation.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  All
 *    device work is enqueued on it, asynchronously.
 *  - Matrices are row-major.  Row i of G and Bᵀ, and column i of Aᵀ, belong to
 *    points[i] (caller order honoured; drivers pass canonical order = finite points
 *    ascending, +INFINITY last).
 */
#ifndef WINO_H_
#define WINO_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  WINO_OK = 0,
  WINO_E_INVALID_ARG = 1,      /* NULL pointer, m < 1, r < 1, n_cand < 0, dims not 1|2, pad < 0 ... */
  WINO_E_BAD_SHAPE = 2,        /* n != m + r - 1; empty output (H + 2 pad < r)                       */
  WINO_E_DUPLICATE_POINTS = 3, /* two finite points compare equal (exact ==; +0 == -0)               */
  WINO_E_INF_NOT_LAST = 4,     /* +INFINITY anywhere but the last slot, or -INFINITY anywhere        */
  WINO_E_NONFINITE_POINT = 5,  /* NaN point                                                          */
  WINO_E_WORKSPACE = 6,        /* workspace NULL or smaller than the *_workspace_bytes() figure      */
  WINO_E_CUDA = 7,             /* CUDA launch / configuration error (detail in wino_last_error())    */
  WINO_E_UNSUPPORTED = 8       /* (dims, m, r) without a compiled kernel (see wino_supported())      */
} wino_status;

#define WINO_MAX_N 16 /* n = m + r - 1 accepted by wino_points_to_matrices */

/* Error statistics ("L1 norm ... between the output of each type of convolution
 * and a normal convolution using double precision"; per element, reading R10).  fp64,
 * per scored unit (candidate, or layer):
 *   sums[5] = { Σ|e|, Σe², Σ|y_ref|, n_scored, n_nonfinite },  maxs[2] = { max|e|, max|y_ref| }
 * with e = RN64((double)y32 − y64) for every output.  A non-finite e only increments
 * n_nonfinite (it is excluded from Σ|e|, Σe², max|e|, n_scored); Σ|y_ref| and max|y_ref|
 * describe the reference and run over every output (reading R16).
 * Calls ACCUMULATE (sums +=, maxs = max) so buffers can be summed over
 * calls and all-reduced over ranks; the caller zero-initialises them.
 * Mean absolute error = sums[0] / sums[3]. */
#define WINO_SUMS 5
#define WINO_MAXS 2

/* Sweep flags. */
#define WINO_SWEEP_NOFMA 1u /* paper arithmetic acc = RN(acc + RN(a*b)) instead of fmaf chains (R13) */
/* Huffman evaluation order of every transform dot product ("Huffman tree evaluation
 * order"; reading R21): products RN(coef*x) of the non-zero coefficients
 * summed along a Huffman tree over |coef| (ties: leaves in index order, then older nodes);
 * Hadamard product RN(u*v).  Overrides WINO_SWEEP_NOFMA.  Compiled for F(m,3), m = 2..8
 * (the paper's T7/T8 sizes), in 1D and 2D; other shapes return WINO_E_UNSUPPORTED. */
#define WINO_SWEEP_HUFFMAN 2u
/* Mixed precision ("double precision floating point for the transforms and single
 * precision for Hadamard product"; reading R22): the transforms in fp64 with the
 * fp64 (R64) matrices (ascending fma chains), U and V rounded to fp32, M = RN32(u*v), the
 * output transform in fp64 rounded to fp32.  Compiled for F(2,3), F(4,3), F(6,3) in 1D and
 * 2D; cannot be combined with WINO_SWEEP_HUFFMAN (WINO_E_INVALID_ARG). */
#define WINO_SWEEP_MIXED 4u

const char* wino_status_string(int status);
const char* wino_last_error(void);
/* 1 if a kernel for (dims, m, r) is compiled into this library, else 0. */
int wino_supported(int dims, int m, int r);

/* (1) Points -> transform matrices.  Host only, synchronous, pure, thread-safe.
 *
 * Defines (§4.1; §4.2 modified algorithm):
 *   Aᵀ[p][i] = αᵢ^p (m x n), G[i][q] = αᵢ^q / Nᵢ with Nᵢ = ∏_{j≠i}(αᵢ − αⱼ) (n x r; the
 *   scaling factor is DIVIDED, reading R1), Bᵀ row i = ascending coefficients of
 *   Mᵢ(x) = ∏_{j≠i}(x − αⱼ) (n x n).  If points[n-1] == +INFINITY (modified Toom-Cook):
 *   the products run over the n-1 finite points, G's last row is [0..0 1], Aᵀ's last
 *   column is [0..0 1]ᵀ, Bᵀ's last row holds the coefficients of M′(x) = ∏ⱼ(x − αⱼ) and
 *   its last column is [0..0 1]ᵀ (reading R4).
 * Arithmetic: the fixed fp64 recipe R64: every entry is bit-identical
 * to the oracle's.  points: HOST double[n], n = m + r − 1 ≤ WINO_MAX_N.
 * AT: HOST double[m*n], G: HOST double[n*r], BT: HOST double[n*n] (caller-allocated,
 * fully overwritten on success, untouched on error).
 * Errors: INVALID_ARG, BAD_SHAPE, DUPLICATE_POINTS, INF_NOT_LAST, NONFINITE_POINT,
 * UNSUPPORTED (n > WINO_MAX_N). */
int wino_points_to_matrices(int m, int r, const double* points, int n,
                            double* AT, double* G, double* BT);

/* (2) fp32 Winograd convolution layer F(m x m, r x r), stride 1, symmetric zero padding
 * `pad`, no bias (eq:conv P:112 read as valid cross-correlation, R3; eq:conv_2d P:181;
 * channel sum in the Winograd domain).
 *   x: DEVICE float[N][C][H][W]  w: DEVICE float[K][C][r][r]
 *   y: DEVICE float[N][K][Ho][Wo], Ho = H + 2 pad − r + 1, Wo = W + 2 pad − r + 1
 *   points: HOST double[m + r − 1] (rules of (1)); the fp32 matrices are RN32 of (1).
 *   workspace: DEVICE, >= wino_conv2d_workspace_bytes(...) bytes, 256-byte aligned.
 *   d_sums / d_maxs: DEVICE double[WINO_SUMS] / double[WINO_MAXS], or both NULL.  When
 *   non-NULL every output is also scored against the fp64 direct convolution of the same
 *   fp32 x, w and the statistics are ACCUMULATED into them.
 * Arithmetic (the parity semantics, DESIGN.md §2.3 "F32-FMA"): each dot product is an
 * ascending fmaf chain from +0; 2D transforms left product first; the channel sum is one
 * ascending-c fmaf chain per (k, tile, Winograd position), no split, no TF32.
 * Output is bit-identical to the oracle's O5 layer.  N == 0 or K == 0 (empty output) is a
 * successful no-op (nothing enqueued, statistics untouched); C, H, W >= 1 are required.
 * Asynchronous on `stream` and stream-ordered: the kernels of one call form a
 * programmatic-dependent-launch chain on `stream` (n <= 8), or the filter transform runs on
 * a library-owned side stream (one per host thread and device) forked from and joined back
 * to `stream` with events (n > 8, the variants of (2c), the timing hook on,
 * WINO_LAYER_NO_PDL=1); C <= 4 layers run the transforms and the contraction in one fused
 * kernel (same bits).  wino_conv2d_workspace_bytes() is large enough for every variant of
 * (2c) as well. */
size_t wino_conv2d_workspace_bytes(int N, int C, int H, int W, int K, int r, int pad, int m);
/* Diagnostic: which contraction kernel this shape runs in the parity path (2): the CTA tile
 * as 1000 * k_rows + t_cols (128128, 64128 when K <= 64, 128064 when the narrow tile needs
 * fewer waves), 1 for the fused C <= 4 kernel, 0 for invalid or unsupported
 * arguments.  Host only; the tests use it to make sure every variant is exercised. */
int wino_conv2d_gemm_tile(int N, int C, int H, int W, int K, int r, int pad, int m);
int wino_conv2d_fp32(const float* x, const float* w, float* y,
                     int N, int C, int H, int W, int K, int r, int pad, int m,
                     const double* points, void* workspace, size_t workspace_bytes,
                     double* d_sums, double* d_maxs, void* stream);

/* (2c) wino_conv2d_fp32 with variant flags (NEXT row N3, reported separately):
 *   WINO_CONV_TF32: the channel contraction runs on the 5th-generation tensor cores
 *   (tcgen05.mma kind::tf32, accumulator in tensor memory).  TF32 keeps 10 mantissa bits of
 *   each operand, so this variant does NOT have the parity semantics above; its error is
 *   what the scored statistics measure.  Same arguments and workspace as (2). */
#define WINO_CONV_TF32 1u
/*   WINO_CONV_3XTF32: split-precision contraction on the same tensor cores: each operand is
 *   x = hi + lo (hi = tf32(x), lo = tf32(x - hi)) and M += lo*hi + hi*lo + hi*hi with fp32
 *   accumulation, recovering ~fp32 accuracy (not bit-identical to the parity path).  Takes
 *   precedence over WINO_CONV_TF32. */
#define WINO_CONV_3XTF32 2u
/*   WINO_CONV_SCORE_PER_IMAGE: with d_sums / d_maxs non-NULL, the statistics are kept per
 *   image: d_sums DEVICE double[N][WINO_SUMS], d_maxs DEVICE double[N][WINO_MAXS] (row n =
 *   image n, accumulated).  Each image's statistics depend only on that image, so a
 *   batch-sharded network reduces them over images in a fixed order and gets
 *   results independent of the number of ranks.  Combinable with the other flags. */
#define WINO_CONV_SCORE_PER_IMAGE 4u
int wino_conv2d_fp32_ex(const float* x, const float* w, float* y,
                        int N, int C, int H, int W, int K, int r, int pad, int m,
                        const double* points, void* workspace, size_t workspace_bytes,
                        double* d_sums, double* d_maxs, unsigned flags, void* stream);

/* (2d) The layer with the network glue of configs[4] fused into its output transform:
 *   act = maxpool_pool(ReLU(conv)), pool 1 | 2 (2 x 2 window, stride 2, floor), DEVICE
 *   float[N][K][Ho/pool][Wo/pool]; y: DEVICE float[N][K][Ho][Wo] conv output, or NULL when
 *   neither the scoring (d_sums) nor the caller needs it (then y is never materialised).
 *   For even m the ReLU / pool run in the output-transform epilogue (a pooling window never
 *   straddles two m x m tiles); odd m with pool 2 needs y and runs kernel (2b) after it.
 *   ReLU and max are exact: act equals wino_relu_pool_fp32(y) bit for bit.  Other arguments,
 *   flags and errors as (2c); INVALID_ARG also for act == NULL, pool not 1|2, or y == NULL
 *   where it is required. */
int wino_conv2d_relu_pool_fp32(const float* x, const float* w, float* y, float* act,
                               int N, int C, int H, int W, int K, int r, int pad, int m,
                               const double* points, void* workspace, size_t workspace_bytes,
                               double* d_sums, double* d_maxs, int pool, unsigned flags, void* stream);

/* (2b) Network glue for BASELINE.json configs[4] (VGG-16 "ReLU + 2x2 maxpool"):
 *   y[n][c][h][w] = max(0, max_{a,b < pool} x[n][c][pool h + a][pool w + b]), pool 1 | 2
 *   (2 x 2 window, stride 2, floor).  x: DEVICE float[N][C][H][W], y: DEVICE
 *   float[N][C][H/pool][W/pool].  Exact (no rounding).  Asynchronous on `stream`. */
int wino_relu_pool_fp32(const float* x, float* y, int N, int C, int H, int W, int pool, void* stream);

/* (3) Error sweep over candidate point sets on ONE device (P:465 error protocol; P:472
 * sweep; the multi-GPU driver shards candidates over ranks and all-reduces the stats).
 *   dims 1|2; point_sets: HOST double[n_cand][n] (each row obeys (1)).
 *   d_tiles: DEVICE float[n_tiles][n^dims], g_tiles: DEVICE float[n_tiles][r^dims]
 *   (row-major n x n / r x r tiles; the SAME tiles score every candidate, O9), both
 *   16-byte aligned (vector loads; else WINO_E_INVALID_ARG).
 *   d_sums: DEVICE double[n_cand][WINO_SUMS], d_maxs: DEVICE double[n_cand][WINO_MAXS]
 *   (ACCUMULATED for accepted candidates).  cand_status: HOST int[n_cand] out, per-candidate
 *   wino_status of (1); a rejected candidate does not fail the call and its statistics rows
 *   are OVERWRITTEN with NaN (so a caller can never read a silent 0/0 mean).
 *   workspace: DEVICE, >= wino_error_sweep_workspace_bytes(...), 256-byte aligned.
 *   flags: WINO_SWEEP_*.
 * Every output of every tile is scored against the fp64 direct correlation of the tile.
 * A candidate whose outputs are not all finite is scored exactly per output (n_nonfinite
 * counts the non-finite e over the real tiles).  Asynchronous on `stream` (host matrix
 * construction happens before the launch).  n_tiles == 0: accepted rows untouched. */
size_t wino_error_sweep_workspace_bytes(int dims, int m, int r, int n_cand, int64_t n_tiles);
int wino_error_sweep(int dims, int m, int r, const double* point_sets, int n_cand,
                     const float* d_tiles, const float* g_tiles, int64_t n_tiles,
                     double* d_sums, double* d_maxs, int* cand_status,
                     void* workspace, size_t workspace_bytes, unsigned flags, void* stream);

/* (3b) The same sweep with the fp32 outputs written out: the PRODUCTION kernels of (3)
 * (the output store is a run-time branch of the same code, not a separate build), used for
 * per-element parity against the oracle.
 *   d_y: DEVICE float[n_cand][n_tiles][m^dims]; rows of rejected candidates are untouched.
 *   d_sums / d_maxs: as in (3), or both NULL (statistics computed in the workspace only).
 *   workspace: DEVICE, >= wino_error_sweep_workspace_bytes(...). */
int wino_sweep_outputs(int dims, int m, int r, const double* point_sets, int n_cand,
                       const float* d_tiles, const float* g_tiles, int64_t n_tiles,
                       float* d_y, double* d_sums, double* d_maxs, int* cand_status,
                       void* workspace, size_t workspace_bytes, unsigned flags, void* stream);

/* Huffman-order sweeps (WINO_SWEEP_HUFFMAN) run either the shared-memory interpreter
 * kernel (per-candidate programs in the kernel parameters) or, per class of candidates
 * with identical per-row Huffman programs, a kernel generated from those programs and
 * compiled at run time with NVRTC for sm_100a (every tree as straight-line register code;
 * bit-identical outputs, statistics equal up to fp64 summation order).  mode: 0 = auto
 * (run-time kernels for sweeps of >= 16384 tiles when NVRTC loads), 1 = always, 2 = never.
 * Process-wide; returns the previous mode.  Compiled kernels are cached for the process
 * (wino_huffman_jit_classes() = how many).  A failed compilation in a call that uses them
 * returns WINO_E_CUDA with NVRTC's log in wino_last_error(). */
int wino_huffman_jit_mode(int mode);
int wino_huffman_jit_classes(void);
/* Diagnostic (host only, no GPU needed): generate and NVRTC-compile the Huffman-order kernel
 * of the class of one HOST point set [m + r - 1]; *cubin_bytes = the sm_100a cubin size.
 * Returns WINO_OK, a point-set status, or WINO_E_CUDA (log in wino_last_error()). */
int wino_huffman_jit_compile_check(int dims, int m, int r, const double* points, size_t* cubin_bytes);

/* Number of kernel launches the last successful call on this thread enqueued
 * (for bench.py's gpu_launches count). */
int wino_last_launch_count(void);

/* Kernel timing hook (profiling / bench.py roofline).  While enabled, every launch is
 * bracketed by two cudaEvents recorded on its own stream and filed under its kernel
 * family: "sweep1d", "sweep2d", "sweep_huffman", "sweep_mixed", "sweep_refs1d", "sweep_refs2d", "sweep_finalize",
 * "layer_filter", "layer_input", "layer_gemm", "layer_gemm_tf32", "layer_gemm_3xtf32", "layer_output", "layer_score",
 * "layer_score_finalize", "relu_pool".  Exception: the candidate-chunk launches of one sweep call
 * ("sweep1d", "sweep2d", "sweep_huffman", "sweep_mixed") form a programmatic-dependent-launch
 * chain (each chunk may start while the previous drains); the chain is bracketed by ONE event
 * pair and counts as its number of launches.  wino_timing_read() synchronises on the recorded
 * events and returns the summed milliseconds and launch count of one family since the last reset.
 * Returns the previous enable state / a wino_status. */
int wino_timing_enable(int enable);
void wino_timing_reset(void);
int wino_timing_read(const char* family, double* total_ms, int* launches);

#ifdef __cplusplus
}
#endif
#endif /* WINO_H_ */
