/*
 * hsk.h -- C ABI of libhsk.so, the sm_100a sketch engine.
 *
 * Drop-in boundary for the sketch hot path of hsskit (arXiv 2302.01977
 * reference, /root/reference/pkg/src/hsskit/sketching.py).  Each entry point
 * replaces one reference function; the Python host mirror
 * (paper_2302_01977_b200/sketching.py) binds them with ctypes exactly as the
 * reference's own operator API would.
 *
 * Conventions
 *  - All matrix pointers are DEVICE pointers owned by the caller.
 *  - Matrices are column-major (Fortran order, as `_buffer_of` produces,
 *    sketching.py:76-79) with an explicit leading dimension.
 *  - `A` is rows x cols with leading dimension lda >= rows.
 *      trans == 0:  S  = A   * R^T   needs cols == n, S is rows x d
 *                   (reference apply_right, sketching.py:431-442)
 *      trans == 1:  S' = A^T * R^T   needs rows == n, S is cols x d
 *                   (reference apply_right_transposed, sketching.py:445-457)
 *  - Output S is column-major with leading dimension lds; the d sketch
 *    columns are written at column offset col0, so adaptive appends land in
 *    a preallocated capacity-d_max buffer without re-reading old columns
 *    (hss_compress.py:168-182).
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Launches are
 *    stream-ordered and return immediately.
 *  - Results are deterministic: fixed reduction order, no floating-point
 *    atomics.
 *  - Return value: HSK_OK or a negative status; hsk_last_error() gives the
 *    message.  Status classes mirror the reference's exceptions:
 *    HSK_EINVAL -> ValueError, HSK_ERANGE -> IndexError,
 *    HSK_ECUDA/HSK_ENODEV -> RuntimeError.
 */
#ifndef HSK_H
#define HSK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HSK_ABI_VERSION 1

#if defined(__GNUC__)
#define HSK_API __attribute__((visibility("default")))
#else
#define HSK_API
#endif

#define HSK_OK      0
#define HSK_EINVAL -1   /* bad shape / parameter          -> ValueError   */
#define HSK_ERANGE -2   /* index out of range             -> IndexError   */
#define HSK_ECUDA  -3   /* CUDA runtime / launch failure  -> RuntimeError */
#define HSK_ENODEV -4   /* no sm_100 device               -> RuntimeError */

HSK_API int hsk_abi_version(void);

/* Tuning knobs (HSK_SJLT_* / HSK_GAUSS_CFG environment variables, see
 * DESIGN.md) are read once, on first use; this re-reads them after the
 * environment changed in-process (A/B tools and tests).  No reference
 * counterpart. */
HSK_API int hsk_tuning_reload(void);

/* Number of hsk_tuning_reload() calls so far.  An SJLT plan's geometry (chunk
 * size, tile layout) depends on the knobs, so a plan must be applied under the
 * knobs it was built with: callers that cache plans rebuild them when this
 * changes (device.block_state does).  No reference counterpart. */
HSK_API int hsk_tuning_generation(void);

/* Copies the calling thread's last error message into buf (NUL-terminated);
 * returns its full length. */
HSK_API int hsk_last_error(char *buf, size_t len);

/* sm_count, compute capability and L2 size of the current device. */
HSK_API int hsk_device_info(int *sm_count, int *cc_major, int *cc_minor, int64_t *l2_bytes);

/* ------------------------------------------------------------------ SJLT
 * Replaces SjltBlock._build_storage (sketching.py:292-320): the reference
 * builds index-only CSR/CSC views of B+ and B- (PAPER.md:864-901); the GPU
 * plan is the same pattern re-blocked for the kernel: per k-chunk of the
 * input index, the entries sorted by bucket (stable in (k, t)), each entry a
 * 32-bit word (sign in bit 31 | bucket within its warp group << 24 | tile
 * offset of k), every group of buckets one consumer warp owns closed by a
 * terminator word, plus per-chunk u32 group starts (one sub-plan per
 * direction).
 *   pos: n x alpha int32 (reference `_pos`), values in [0, d)
 *   sgn: n x alpha int8  (reference `_signs`), values +-1
 * hsk_sjlt_plan_bytes gives the size of the device buffer `plan`. */
HSK_API int64_t hsk_sjlt_plan_bytes(int64_t n, int32_t d, int32_t alpha);
HSK_API int hsk_sjlt_plan_build(const int32_t *pos, const int8_t *sgn, int64_t n, int32_t d,
                        int32_t alpha, void *plan, int64_t plan_bytes, void *stream);

/* Chunked patterns (flags = HSK_SJLT_CHUNKED): the block construction
 * (SjltBlock.__init__, sketching.py:246-250) places entry t of every input
 * index in chunk t of d/alpha buckets, pos(k,t) in [t*d/alpha, (t+1)*d/alpha).
 * With d/alpha = 8 and d a multiple of 64 (C3: alpha = 8 increments of 64) the
 * plan pairs the chunks: one consumer warp owns two chunks and reads each
 * element once for both (alpha/2 tile reads per element instead of alpha).
 * Other shapes ignore the flag.  For paired shapes plan_build verifies the
 * chunk property on the device and returns HSK_EINVAL if it fails (it then
 * synchronises `stream` once); plan_bytes / plan_build / apply must all get
 * the same flags. */
#define HSK_SJLT_CHUNKED 1
HSK_API int64_t hsk_sjlt_plan_bytes_ex(int64_t n, int32_t d, int32_t alpha, int32_t flags);
HSK_API int hsk_sjlt_plan_build_ex(const int32_t *pos, const int8_t *sgn, int64_t n, int32_t d,
                           int32_t alpha, int32_t flags, void *plan, int64_t plan_bytes,
                           void *stream);
HSK_API int hsk_sjlt_apply_ex(const double *A, int64_t rows, int64_t cols, int64_t lda,
                      int32_t trans, const void *plan, int64_t n, int32_t d, int32_t alpha,
                      int32_t flags, double scale, double *S, int64_t lds, int64_t col0,
                      void *stream);

/* Replaces SjltBlock.apply_right (trans 0, sketching.py:322-332) and
 * SjltBlock.apply_right_transposed (trans 1, sketching.py:334-351):
 * S[:, col0 + j] = scale * sum_k sgn(k,t) A[:, k]  over (k,t) with pos = j. */
HSK_API int hsk_sjlt_apply(const double *A, int64_t rows, int64_t cols, int64_t lda, int32_t trans,
                   const void *plan, int64_t n, int32_t d, int32_t alpha, double scale,
                   double *S, int64_t lds, int64_t col0, void *stream);

/* -------------------------------------------------------------- Gaussian
 * Replaces GaussianBlock.apply_right (buf @ matrix.T) and
 * apply_right_transposed ((matrix @ buf).T), sketching.py:134-138.
 *   R: the reference `matrix`, d x n row-major (== R^T column-major, ld n).
 * FP64 DMMA (mma.sync m8n8k4) tensor-core contraction. */
HSK_API int hsk_gauss_apply(const double *A, int64_t rows, int64_t cols, int64_t lda, int32_t trans,
                    const double *R, int64_t n, int32_t d, double *S, int64_t lds,
                    int64_t col0, void *stream);

/* FP64 tensor-pipe peak probe (no reference counterpart): sm_count * 2 CTAs of
 * 8 warps, each `iters` x 8 independent DMMA.8x8x4; hsk_dmma_probe_flops gives
 * the flops of one launch.  Time it with events for the FP64 roofline
 * denominator of hsk_gauss_apply (bench.py).  scratch: one device double. */
HSK_API int64_t hsk_dmma_probe_flops(int64_t iters);
HSK_API int hsk_dmma_probe(int64_t iters, double *scratch, void *stream);

/* ------------------------------------------------------------------ SRHT
 * Replaces SrhtBlock._transform (sketching.py:162-176):
 *   S[r, col0 + t] = scale * FWHT_npad(pad(x_r) .* signs)[sample[t]]
 * for each row x_r of A (trans 0) or column (trans 1).
 *   signs: n_pad doubles (+-1), sample: d int64 in [0, n_pad) (with
 *   replacement, as drawn by the reference, sketching.py:158-159). */
HSK_API int hsk_srht_apply(const double *A, int64_t rows, int64_t cols, int64_t lda, int32_t trans,
                   const double *signs, int64_t n, int64_t n_pad, const int64_t *sample,
                   int32_t d, double scale, double *S, int64_t lds, int64_t col0,
                   void *stream);

/* Replaces fwht (sketching.py:100-112) on `rows` contiguous rows of length
 * n (a power of two) in place; normalize != 0 scales by 1/sqrt(n). */
HSK_API int hsk_fwht(double *X, int64_t rows, int64_t n, int32_t normalize, void *stream);

/* ------------------------------------------------- synthetic generators
 * Benchmark inputs of BASELINE.json (no reference counterpart: hsskit's
 * matgen.py has neither matrix).  Write the block rows [row0,row0+nrows) x
 * cols [col0, col0+ncols) of the n x n matrix into A (column-major, lda).
 * Gaussian kernel: A_ij = exp(-|x_i - x_j|^2 / (2 h^2)) + diag * (i == j),
 *   pts is n x dim row-major (device).
 * Toeplitz-sine:   A_ij = 1/(1 + |i-j|) + 0.1 sin(i + 2j) / n.            */
HSK_API int hsk_gen_gauss_kernel(const double *pts, int64_t n, int32_t dim, double h, double diag,
                         int64_t row0, int64_t nrows, int64_t col0, int64_t ncols,
                         double *A, int64_t lda, void *stream);
HSK_API int hsk_gen_toeplitz_sin(int64_t n, int64_t row0, int64_t nrows, int64_t col0, int64_t ncols,
                         double *A, int64_t lda, void *stream);

/* B = A^T: A rows x cols column-major (lda), B cols x rows column-major (ldb),
 * both device, not overlapping.  The adaptive sketch keeps A^T once so every S' increment runs
 * as S = A^T R^T on conflict-free tiles (adaptive.DeviceSketch). */
HSK_API int hsk_transpose(const double *A, int64_t rows, int64_t cols, int64_t lda, double *B,
                          int64_t ldb, void *stream);

/* *flag (one int32, DEVICE memory) = 1 if the n x n column-major A (lda) is not
 * bitwise symmetric, else 0 (stream-ordered; read it after a sync).  An adaptive
 * sketch of a symmetric A gets S' = A^T R^T = A R^T = S, bit for bit. */
HSK_API int hsk_is_symmetric(const double *A, int64_t n, int64_t lda, int32_t *flag, void *stream);

/* Streams `bytes` of scratch (device) to evict L2 between timed launches. */
HSK_API int hsk_l2_flush(void *scratch, int64_t bytes, void *stream);

/* ------------------------------------------ peer memory (multi-GPU S')
 * Row-sharded S' = A^T R^T (BASELINE.json C5): the reference sums per-shard
 * partials with a collective; here each rank's S' kernel writes destination
 * block q directly into rank q's receive slot through an IPC mapping (the
 * transfer rides on the kernel's epilogue stores), then the owner sums its
 * slots in rank order.  Handles are HSK_IPC_HANDLE_BYTES opaque bytes. */
#define HSK_IPC_HANDLE_BYTES 64
HSK_API int hsk_ipc_alloc(int64_t bytes, void **ptr, void *handle);
HSK_API int hsk_ipc_free(void *ptr);
HSK_API int hsk_ipc_open(const void *handle, void **ptr);
HSK_API int hsk_ipc_close(void *ptr);
/* out(r, c) = sum over g = 0..nslices-1 (in order) of base[g*stride + c*ld + r];
 * column-major rows x cols slices, deterministic. */
HSK_API int hsk_sum_slices(const double *base, int32_t nslices, int64_t stride, int64_t rows,
                   int64_t cols, int64_t ld, double *out, int64_t ldo, void *stream);

/* ------------------------------------------ HSS sweep dense kernels
 * Column-pivoted Householder QR truncated at the numerical rank: replaces
 * scipy.linalg.qr(S, mode="r", pivoting=True) (LAPACK dgeqp3) and the rank
 * count of interpolative_decomposition (dense_kernels.py:54-82).
 *   M: m x n column-major (ldm), OVERWRITTEN.  Pivoting as LAPACK's
 *   dgeqp2/dlaqp2 (first position of maximal partial column norm; dlarfg
 *   reflectors; dlaqp2 norm downdates).  Stops at the first step j with
 *   |R_jj| < max(eps_abs, eps_rel |R_00|) (an all-zero M has rank 0).
 *   perm: n int64 (perm[i] = column at pivot position i); R: the first
 *   *rank rows of R in pivot order, column-major (ldr >= max(min(m,n),1));
 *   rank: ONE int32 in DEVICE memory (stream-ordered; read it after a sync).
 *   work: hsk_pqr_work_bytes(m, n) bytes of device scratch.
 * One cooperative launch (co-resident CTAs, a grid barrier per step). */
HSK_API int64_t hsk_pqr_work_bytes(int64_t m, int64_t n);
HSK_API int hsk_pqr(double *M, int64_t m, int64_t n, int64_t ldm, double eps_rel, double eps_abs,
                    int64_t *perm, double *R, int64_t ldr, int32_t *rank, void *work,
                    int64_t work_bytes, void *stream);

/* Strided async copy of `height` rows of `width` bytes (pitches in bytes);
 * kind 1 = host -> device, 2 = device -> host.  Used to stream row slabs of a
 * pinned host matrix through the kernels (copy / compute overlap). */
HSK_API int hsk_memcpy2d(void *dst, int64_t dpitch, const void *src, int64_t spitch, int64_t width,
                 int64_t height, int32_t kind, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* HSK_H */
