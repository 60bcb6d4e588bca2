/*
 * dash_b200.h -- C ABI of the B200-native DASH (dual-way streaming PARAFAC2)
 * per-update step.  Built as paper_2305_18376_b200/libdash_b200.so (sm_100a).
 *
 * Conventions (all entry points):
 *   - every array argument is a DEVICE pointer unless its name ends in _host;
 *     row-major, FP64 ("f64" suffix); the caller (torch) owns all of them;
 *   - the library owns only the workspace arena inside a dash_ctx;
 *   - work is enqueued on the given cudaStream_t (passed as void*) and is
 *     stream-ordered; nothing synchronises the host except
 *     dash_ctx_status(), which waits for the stream and reads the error slot;
 *   - return value: 0 on success, a DASH_E* code otherwise (launch / shape
 *     errors are reported immediately, numerical failures via
 *     dash_ctx_status() because they are only known on the device).
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/p2stream):
 *   dash_update_f64         StreamState.update pass loop     stream.py:251-370
 *   dash_group_update_f64   numba group_update seam          _kernels.py:62-149
 *   dash_ridge_solve_f64    ridge_solve (V solve, update_v)   linalg.py:25-45,
 *                                                             stream.py:158-160,346
 *   dash_init_helpers_f64   init_helpers                      stream.py:56-82
 *   dash_local_error_f64    local_error / slice_error         evaluate.py:93-118,
 *                                                             anomaly.py:23-42
 *   dash_als_sweep_f64      parafac2_als sweep (initialize)    als.py:102-201
 *   dash_update_f32 / dash_update_pass_begin_f32 / dash_local_error_f32
 *                           the same update / fitness with the streamed data
 *                           in FP32 (north_star's optional FP32 mode; the
 *                           reference has FP64 only)
 */
#ifndef DASH_B200_H
#define DASH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DASH_OK 0
#define DASH_E_ARG 1        /* bad shape / null pointer / unsupported rank   */
#define DASH_E_CUDA 2       /* a CUDA launch or allocation failed            */
#define DASH_E_SINGULAR 3   /* a ridge system was singular (LU zero pivot)  */
#define DASH_E_NONFINITE 4  /* a solve produced a non-finite value          */

#define DASH_MAX_RANK 64      /* update path (dash_update*, group_update)      */
#define DASH_MAX_RANK_ALS 32  /* ALS sweep, init_helpers, ridge_solve           */

typedef struct dash_ctx dash_ctx;

/* Create / destroy a context bound to the current CUDA device. */
int dash_ctx_create(dash_ctx **out);
void dash_ctx_destroy(dash_ctx *ctx);

/* Wait for `stream`, then report the first numerical failure since the last
 * call: returns DASH_OK or DASH_E_SINGULAR / DASH_E_NONFINITE, with
 * *fail_slice_host = batch position of the failing slice (-1 = the V solve).
 * Clears the slot. */
int dash_ctx_status(dash_ctx *ctx, void *stream, int64_t *fail_slice_host);

/* Kernel launches issued by the last dash_update_f64 call (for bench.py's
 * gpu_launches figure). */
int dash_ctx_last_launches(const dash_ctx *ctx);

/* Host helper (no device work): row_ptr[0] = 0, row_ptr[m+1] = row_ptr[m] +
 * counts[m] for m < M (row_ptr may be pinned memory that is then copied to
 * the device), *N_out = total rows.  DASH_E_ARG on a negative count. */
int dash_host_row_ptr(const int64_t *counts, int64_t M, int64_t *row_ptr, int64_t *N_out);

/* Batch index staging (the host half of stream.py:282-298, the reference's
 * per-update grouping / staging): a ring of caller-owned slots, each a pinned
 * host block and a device block of `cap` bytes.  dash_stage_meta packs
 *   row_ptr (M+1) i64 | state_row (M) i32, padded to 8 bytes | is_new (M) u8
 * for a batch of M_old existing slices (state rows `existing_rows`) followed by
 * L new slices (state rows K_base ..) into the next slot's pinned block, copies
 * it to the slot's device block on the context's side stream (overlapping the
 * previous update's kernels) and makes `stream` wait for that copy; with
 * keep_dev != NULL the packed block is also copied there (device to device, on
 * `stream`) for the U history.  dash_stage_release records, on `stream`, that
 * the update which read the last staged slot has been issued in full -- the slot's
 * device block is rewritten only after that point; the final dash_update_pass_finish
 * of an update (and so dash_update_f64 / _f32) does the same, so callers that run
 * the staged batch through those entry points need not call it.  The host blocks only when
 * the ring wraps onto a copy still in flight. */
typedef struct dash_staged {
    int64_t N;               /* total rows of the batch */
    int32_t M;               /* slices */
    int32_t slot;            /* ring slot used */
    const void *row_ptr;     /* device, int64 (M+1) */
    const void *state_row;   /* device, int32 (M) */
    const void *is_new;      /* device, uint8 (M) */
    const void *row_ptr_host;/* pinned, valid until the ring wraps */
    int64_t nbytes;          /* size of the packed block */
} dash_staged;
int dash_meta_ring_set(dash_ctx *ctx, int32_t nslots, void *const *pinned, void *const *device, int64_t cap);
int dash_stage_meta(dash_ctx *ctx, void *stream, const int64_t *counts, int32_t M_old, const int32_t *existing_rows,
                    int32_t L, int32_t K_base, void *keep_dev, dash_staged *out);
int dash_stage_release(dash_ctx *ctx, void *stream);

/* Kernel path chosen for the last update (for benchmarks): bit 0 = streaming
 * (TMA-ring) GEMMs, bit 1 = tensor-map boxes (k_xv3 / k_fgemm3 or the FP32
 * variants), bit 2 = fused big-slice path (k_bigx: big-slice rows read once). */
#define DASH_PATH_STREAM 1
#define DASH_PATH_TMA 2
#define DASH_PATH_BIGX 4
#define DASH_PATH_SMALLX 8  /* bit 3: fused small-slice kernel (k_smallx: small-slice rows read once for XV,
                               re-read from L2 for F; no XV / U o w round trips) */
int dash_ctx_path_flags(const dash_ctx *ctx);

/* Number of ridge systems that needed the LU fallback (Cholesky failed or a
 * non-finite solution) since the last reset; syncs `stream`. */
int dash_ctx_fallbacks(dash_ctx *ctx, void *stream, int32_t reset);

/* One update batch in CSR form: slice m (batch position) owns rows
 * [row_ptr[m], row_ptr[m+1]) of X.  Order = UpdateBatch.items() order
 * (tensor.py:166-171): existing slices, then new slices. */
/* Rows per batch are addressed with 32-bit offsets inside the kernels. */
#define DASH_MAX_BATCH_ROWS 2147483647LL

typedef struct {
    const double *X;             /* N x ldx                                    */
    int64_t ldx;                 /* >= J                                        */
    int64_t N;                   /* total new rows                              */
    int32_t M;                   /* slices in the batch                         */
    const int64_t *row_ptr;      /* M+1 (device)                                */
    const int64_t *row_ptr_host; /* M+1 (host copy, used for work planning)     */
    const int32_t *state_row;    /* M: row of W/C/D owned by the slice          */
    const uint8_t *is_new;       /* M: 1 = registered by this batch             */
} dash_batch_f64;

/* FP32 data mode: the same batch with X in single precision (ldx % 4 == 0
 * and a 16-byte aligned X enable the TMA path).  Only the streamed data (X in,
 * U_new out) are FP32; the per-slice state and the factors stay FP64 on the
 * device, and every product / sum inside the kernels is formed in FP64. */
typedef struct {
    const float *X;              /* N x ldx                                    */
    int64_t ldx;
    int64_t N;
    int32_t M;
    const int64_t *row_ptr;
    const int64_t *row_ptr_host;
    const int32_t *state_row;
    const uint8_t *is_new;
} dash_batch_f32;

/* Stream state (StreamState fields, stream.py:196-206).  W/C/D have at least
 * max(state_row)+1 rows.  F, G, V are updated in place. */
typedef struct {
    double *W;   /* K x R        */
    double *C;   /* K x R        */
    double *D;   /* K x R x R    */
    double *V;   /* J x R        */
    double *F;   /* J x R        */
    double *G;   /* R x R        */
    int32_t J;
    int32_t R;
    double forgetting;  /* lambda in (0, 1]                  */
    int32_t passes;     /* ALS passes per update, >= 1       */
} dash_state_f64;

/* One full DASH update (stream.py:251-370): for each pass, U_new for every
 * slice (pre-update V, W; new slices bootstrap W=1, C=0, D=0), c/D
 * accumulation and the S-row (W) solve, F/G accumulation and the V solve.
 * Writes U_out (N x R, batch row order) and v_used_out (J x R, V at the start
 * of the last pass).  W rows are written every pass, C/D rows after the final
 * pass; slices absent from the batch are untouched. */
int dash_update_f64(dash_ctx *ctx, void *stream, const dash_batch_f64 *batch,
                    dash_state_f64 *state, double *U_out, double *v_used_out,
                    double eps);

/* The same update split per pass, for the multi-GPU path: pass_begin runs
 * U / c / D / W for the local slices and writes this rank's fresh sums
 * fg_out = [f (J x R) | g (R x R)] (raw, not yet decayed); the caller
 * all-reduces fg over ranks, then pass_finish forms F = lam F0 + f,
 * G = sym(lam G0 + g) (F0/G0 = state at the start of the update) and solves V.
 * dash_update_f64 == for each pass: pass_begin; pass_finish. */
int dash_update_pass_begin_f64(dash_ctx *ctx, void *stream, const dash_batch_f64 *batch,
                               dash_state_f64 *state, double *U_out, double *v_used_out,
                               double eps, int32_t pass, double *fg_out);
int dash_update_pass_finish_f64(dash_ctx *ctx, void *stream, dash_state_f64 *state,
                                const double *fg, double eps);

/* FP32 data mode of dash_update_f64 / pass_begin: X (batch) and U_out in
 * FP32; state, v_used, fg and all arithmetic FP64.  Results equal the FP64
 * update of the FP32-rounded X up to the final rounding of U_out. */
int dash_update_f32(dash_ctx *ctx, void *stream, const dash_batch_f32 *batch,
                    dash_state_f64 *state, float *U_out, double *v_used_out, double eps);
int dash_update_pass_begin_f32(dash_ctx *ctx, void *stream, const dash_batch_f32 *batch,
                               dash_state_f64 *state, float *U_out, double *v_used_out,
                               double eps, int32_t pass, double *fg_out);

/* Phase timing for benchmarks: when enabled, CUDA events bracket every
 * launch; dash_ctx_phase_ms syncs and returns the summed milliseconds (and
 * launch counts) per phase id since the last call:
 * 0 row_slice (plan), 1 prologue, 2 xv, 3 slices, 4 fgemm, 5 sum_fg, 6 vsolve,
 * 7 big (big-slice kernels: k_big, or k_bigx_pre + k_bigx), 8 big_post (k_bigx_post). */
int dash_ctx_set_profiling(dash_ctx *ctx, int enable);
int dash_ctx_phase_ms(dash_ctx *ctx, double *ms_out, int32_t *count_out, int32_t nphases);

/* The reference's operator seam, same contract as _kernels.group_update:
 * xv (G,I,R), vtv (R,R), s_used (G,R), c_old (G,R), d_old (G,R,R) ->
 * u, us (G,I,R), c_new (G,R), d_new (G,R,R), w (G,R), g_fresh (R,R).
 * *ok_host = 0 when some system needed the LU fallback or failed (the
 * reference's ok=False); outputs are still the fallback solution. */
int dash_group_update_f64(dash_ctx *ctx, void *stream, int32_t G, int32_t I, int32_t R,
                          const double *xv, const double *vtv, const double *s_used,
                          const double *c_old, const double *d_old, double lam, double eps,
                          double *u, double *us, double *c_new, double *d_new, double *w,
                          double *g_fresh, int32_t *ok_host);

/* local_error on an FP32 batch with FP32 U (the FP32 data mode's fitness). */
int dash_local_error_f32(dash_ctx *ctx, void *stream, const dash_batch_f32 *batch,
                         const float *U, const double *W, const double *V, int32_t J,
                         int32_t R, double *slice_err, double *tensor_err);

/* ridge_solve for a batch of systems: x_b = (lhs_b + eps*mean(diag lhs_b) I)^-1 rhs_b,
 * lhs (B,n,n), rhs (B,n,m), x (B,n,m).  n <= DASH_MAX_RANK_ALS. */
int dash_ridge_solve_f64(dash_ctx *ctx, void *stream, int32_t B, int32_t n, int32_t m,
                         const double *lhs, const double *rhs, double *x, double eps);

/* init_helpers over an initial tensor in CSR form (stream.py:56-82):
 * C (K,R) = sum_i (X_k V) o U_k, D (K,R,R) = sym(U_k^T U_k),
 * F (J,R) = sum_k X_k^T (U_k o w_k), G (R,R) = sym(sum_k U_k^T U_k o w_k w_k^T). */
int dash_init_helpers_f64(dash_ctx *ctx, void *stream, const dash_batch_f64 *tensor,
                          const double *U, const double *W, const double *V, int32_t J,
                          int32_t R, double *C, double *D, double *F, double *G);

/* local_error (evaluate.py:93-118): per-slice mean |X_k - (U_k o w_k) V^T|
 * with post-update W, V; slice_err (M), tensor_err (1) = mean over slices. */
int dash_local_error_f64(dash_ctx *ctx, void *stream, const dash_batch_f64 *batch,
                         const double *U, const double *W, const double *V, int32_t J,
                         int32_t R, double *slice_err, double *tensor_err);

/* One sweep of parafac2_als (als.py:153-190) over a tensor in CSR form
 * (row_ptr over K slices, state_row unused): updates V (J,R), H (R,R), W (K,R)
 * in place, writes the sweep's bases Q (N,R) (ALSInfo.projections) and the
 * direct-form loss sum_k ||X_k - Q_k (H o W_k) V^T||^2 to *loss (device). */
int dash_als_sweep_f64(dash_ctx *ctx, void *stream, const dash_batch_f64 *tensor, int32_t J,
                       int32_t R, double *V, double *H, double *W, double *Q, double *loss,
                       double eps);

/* U = Q H for N rows (the final U_k = Q_k H of als.py:191-195). */
int dash_als_project_f64(dash_ctx *ctx, void *stream, int64_t N, int32_t R, const double *Q,
                         const double *H, double *U);

#ifdef __cplusplus
}
#endif
#endif /* DASH_B200_H */
