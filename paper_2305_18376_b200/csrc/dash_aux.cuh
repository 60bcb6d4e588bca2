// Auxiliary entry points around the update step (included by dash_update.cu):
//
//   dash_init_helpers_f64   init_helpers        stream.py:56-82
//   dash_local_error_f64    local_error         evaluate.py:93-118 (+ anomaly.py:23-27)
//   dash_ridge_solve_f64    ridge_solve         linalg.py:25-45
#pragma once

namespace {

// Per-slice c_k, D_k and the G contribution from (XV, U, W) -- init_helpers'
// loop body (stream.py:71-81).  One warp per slice; slot per CTA.
template <int RB, int NW>
__global__ void __launch_bounds__(NW * 32) k_helpers(const int64_t *__restrict__ row_ptr, int M,
                                                     const double *__restrict__ XV, const double *__restrict__ U,
                                                     const double *__restrict__ W, int R, double *__restrict__ C,
                                                     double *__restrict__ D, double *__restrict__ G_slots) {
    constexpr int LD = RB + 1, NP = RB * (RB + 1) / 2, NPC = NP + RB, NPL = (NPC + 31) / 32;
    __shared__ double Us_all[NW][32 * LD];
    __shared__ double Xs_all[NW][32 * LD];
    __shared__ double red[NW][NPC];
    __shared__ int pr_s[NPC], pz_s[NPC];
    const int lane = lane_id(), w = warp_id();
    double *Us = Us_all[w], *Xs = Xs_all[w];
    for (int i = threadIdx.x; i < NPC; i += blockDim.x) {
        int r, z;
        pair_rz(i, RB, r, z);
        pr_s[i] = r;
        pz_s[i] = z;
    }
    __syncthreads();
    double g_loc[NPL];
#pragma unroll
    for (int q = 0; q < NPL; ++q) g_loc[q] = 0.0;
    const int per_cta = (M + gridDim.x - 1) / gridDim.x;
    const int m0 = blockIdx.x * per_cta, m1 = min(M, m0 + per_cta);
    for (int m = m0 + w; m < m1; m += NW) {
        const int64_t r0 = row_ptr[m], r1 = row_ptr[m + 1];
        double gp[NPL];
#pragma unroll
        for (int q = 0; q < NPL; ++q) gp[q] = 0.0;
        for (int64_t c0 = r0; c0 < r1; c0 += 32) {
            const int64_t row = c0 + lane;
            const bool valid = row < r1;
#pragma unroll
            for (int r = 0; r < RB; ++r) {
                Us[lane * LD + r] = (valid && r < R) ? U[row * R + r] : 0.0;
                Xs[lane * LD + r] = (valid && r < R) ? XV[row * R + r] : 0.0;
            }
            __syncwarp();
#pragma unroll
            for (int q = 0; q < NPL; ++q) {
                const int pp = lane + 32 * q;
                if (pp < NPC) {
                    const int a = pr_s[pp], c = pz_s[pp];
                    const double *A = (pp < NP) ? Us : Xs;
                    double acc = gp[q];
                    for (int i = 0; i < 32; ++i) acc = fma(A[i * LD + a], Us[i * LD + c], acc);
                    gp[q] = acc;
                }
            }
            __syncwarp();
        }
#pragma unroll
        for (int q = 0; q < NPL; ++q) {
            const int pp = lane + 32 * q;
            if (pp < NPC) {
                const int r = pr_s[pp], z = pz_s[pp];
                if (r < R && z < R) {
                    if (pp < NP) {
                        D[(int64_t)m * R * R + r * R + z] = gp[q];
                        D[(int64_t)m * R * R + z * R + r] = gp[q];
                        g_loc[q] = fma(gp[q] * W[(int64_t)m * R + r], W[(int64_t)m * R + z], g_loc[q]);
                    } else {
                        C[(int64_t)m * R + r] = gp[q];
                    }
                }
            }
        }
    }
#pragma unroll
    for (int q = 0; q < NPL; ++q)
        if (lane + 32 * q < NPC) red[w][lane + 32 * q] = g_loc[q];
    __syncthreads();
    double *slot = G_slots + (int64_t)blockIdx.x * R * R;
    for (int pp = threadIdx.x; pp < NP; pp += blockDim.x) {
        double acc = 0.0;
        for (int ww = 0; ww < NW; ++ww) acc += red[ww][pp];
        const int r = pr_s[pp], z = pz_s[pp];
        if (r < R && z < R) {
            slot[r * R + z] = acc;
            slot[z * R + r] = acc;
        }
    }
}

// Per-slice mean |X - (U o w) V^T| with post-update W, V; one warp per slice,
// lanes over columns.  V is read through L1 (J x R may exceed shared memory).
template <typename TX>
__global__ void __launch_bounds__(256) k_local_error(const TX *__restrict__ X, int64_t ldx,
                                                     const int64_t *__restrict__ row_ptr,
                                                     const int32_t *__restrict__ state_row, int M,
                                                     const TX *__restrict__ U, const double *__restrict__ W,
                                                     const double *__restrict__ V, int J, int R,
                                                     double *__restrict__ slice_err) {
    const int lane = lane_id();
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    __shared__ double us_s[8][DASH_MAX_RANK];
    double *us = us_s[warp_id()];
    for (int m = gw; m < M; m += nw) {
        const int64_t r0 = row_ptr[m], r1 = row_ptr[m + 1];
        const double *w = W + (int64_t)state_row[m] * R;
        double acc = 0.0;
        for (int64_t row = r0; row < r1; ++row) {
            for (int r = lane; r < R; r += 32) us[r] = (double)U[row * R + r] * w[r];  // R <= 64
            __syncwarp();
            for (int j = lane; j < J; j += 32) {
                double rec = 0.0;
                for (int r = 0; r < R; ++r) rec = fma(us[r], __ldg(V + (int64_t)j * R + r), rec);
                acc += fabs((double)X[row * ldx + j] - rec);
            }
            __syncwarp();
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(FULL_MASK, acc, off);
        if (lane == 0) slice_err[m] = acc / ((double)(r1 - r0) * J);
    }
}

__global__ void k_mean(const double *__restrict__ v, int n, double *__restrict__ out) {
    // fixed-order mean (single thread: n = slices per batch, small)
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double acc = 0.0;
        for (int i = 0; i < n; ++i) acc += v[i];
        *out = n > 0 ? acc / n : 0.0;
    }
}

// Batched ridge_solve: system b = blockIdx.x, lanes over right-hand sides.
// rhs / x entry (r, c) of system b at [b*n*m + r*rs + c*cs] (rs = m, cs = 1 for
// the contiguous (B, n, m) layout; rs = 1, cs = n for the transposed F^T-style
// right-hand sides of the V solves).
template <int RB>
__global__ void __launch_bounds__(32) k_ridge(const double *__restrict__ lhs, const double *__restrict__ rhs,
                                              int n, int m, int64_t rs, int64_t cs, double eps,
                                              double *__restrict__ x, unsigned long long *err) {
    constexpr int LD = RB + 1;
    __shared__ double Ls[RB * LD];
    __shared__ double dinv[RB];
    __shared__ int piv[RB];
    __shared__ double scr[32][LD];
    const int lane = lane_id();
    const int64_t b = blockIdx.x;
    const double *A = lhs + b * n * n;
    double tr = 0.0;
    for (int r = 0; r < n; ++r) tr += A[r * n + r];
    const double sh = eps * (tr / n);
    double row[RB];
#pragma unroll
    for (int z = 0; z < RB; ++z) {
        double v = 0.0;
        if (lane < n && z < n) {
            v = A[lane * n + z];
            if (z == lane) v += sh;
        } else if (z == lane) {
            v = 1.0;
        }
        row[z] = v;
    }
    bool ok = chol_regs<RB>(row, Ls, LD, dinv);
    if (!ok) {
        if (lane == 0) {
            for (int r = 0; r < n; ++r)
                for (int z = 0; z < n; ++z) Ls[r * LD + z] = A[r * n + z] + (r == z ? sh : 0.0);
            if (!lu_factor_serial(Ls, LD, n, piv)) report_error(err, b, DASH_E_SINGULAR);
        }
        __syncwarp();
    }
    for (int c0 = 0; c0 < m; c0 += 32) {
        const int c = c0 + lane;
        const bool valid = c < m;
        double v[RB];
#pragma unroll
        for (int r = 0; r < RB; ++r) v[r] = (valid && r < n) ? rhs[b * n * m + r * rs + c * cs] : 0.0;
        if (ok) {
            chol_solve_lane<RB>(Ls, LD, dinv, v);
        } else {
#pragma unroll
            for (int r = 0; r < RB; ++r)
                if (r < n) scr[lane][r] = v[r];
            if (valid) lu_solve_serial(Ls, LD, n, piv, scr[lane]);
#pragma unroll
            for (int r = 0; r < RB; ++r) v[r] = (r < n) ? scr[lane][r] : 0.0;
        }
        bool fin = true;
#pragma unroll
        for (int r = 0; r < RB; ++r)
            if (valid && r < n) {
                x[b * n * m + r * rs + c * cs] = v[r];
                fin = fin && finite_d(v[r]);
            }
        if (!fin) report_error(err, b, DASH_E_NONFINITE);
        __syncwarp();
    }
}

template <int RB>
static void launch_helpers(cudaStream_t st, int nblocks, const int64_t *row_ptr, int M, const double *XV,
                           const double *U, const double *W, int R, double *C, double *D, double *Gsl) {
    constexpr int NW = RB <= 16 ? 4 : 2;
    k_helpers<RB, NW><<<nblocks, NW * 32, 0, st>>>(row_ptr, M, XV, U, W, R, C, D, Gsl);
}

template <int RB>
static void launch_ridge(cudaStream_t st, int B, const double *lhs, const double *rhs, int n, int m, double eps,
                         double *x, unsigned long long *err) {
    k_ridge<RB><<<B, 32, 0, st>>>(lhs, rhs, n, m, (int64_t)m, (int64_t)1, eps, x, err);
}

}  // namespace

extern "C" {

int dash_init_helpers_f64(dash_ctx *ctx, void *stream, const dash_batch_f64 *t, const double *U, const double *W,
                          const double *V, int32_t J, int32_t R, double *C, double *D, double *F, double *G) {
    if (!ctx || !t || R < 1 || R > DASH_MAX_RANK_ALS || J < 1) return DASH_E_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    ctx->last_launches = 0;
    const int RB = rank_bucket(R);
    const int64_t N = t->N;
    const int M = t->M;
    const int nblocks = std::max(1, std::min(M, ctx->num_sms * 8));
    int64_t nsplit, rps;
    plan_fsplit(ctx, N, J, nsplit, rps);
    if (ensure(ctx->xv, sizeof(double) * std::max<int64_t>(N, 1) * R) ||
        ensure(ctx->row_slice, sizeof(int32_t) * std::max<int64_t>(N, 1)) ||
        ensure(ctx->gslots, sizeof(double) * nblocks * R * R) ||
        ensure(ctx->fslots, sizeof(double) * nsplit * J * R) || ensure(ctx->fsnap, sizeof(double) * J * R) ||
        ensure(ctx->gsnap, sizeof(double) * R * R) || ensure(ctx->scratch, sizeof(int32_t) * std::max(M, 1)))
        return DASH_E_CUDA;
    double *XV = (double *)ctx->xv.p;
    int32_t *row_slice = (int32_t *)ctx->row_slice.p;
    int32_t *ident = (int32_t *)ctx->scratch.p;
    std::vector<int32_t> id(std::max(M, 1));
    for (int i = 0; i < M; ++i) id[i] = i;
    cudaMemcpyAsync(ident, id.data(), sizeof(int32_t) * M, cudaMemcpyHostToDevice, st);
    cudaMemsetAsync(ctx->fsnap.p, 0, sizeof(double) * J * R, st);
    cudaMemsetAsync(ctx->gsnap.p, 0, sizeof(double) * R * R, st);
    dash_batch_f64 b = *t;
    b.state_row = ident;
    if (M > 0 && N > 0) {
        k_row_slice<<<std::min(ctx->num_sms * 4, (M + 7) / 8 + 1), 256, 0, st>>>(t->row_ptr, M, row_slice);
        launch_xv(ctx, st, &b, J, V, R, XV);
        switch (RB) {
            case 4: launch_helpers<4>(st, nblocks, t->row_ptr, M, XV, U, W, R, C, D, (double *)ctx->gslots.p); break;
            case 8: launch_helpers<8>(st, nblocks, t->row_ptr, M, XV, U, W, R, C, D, (double *)ctx->gslots.p); break;
            case 16: launch_helpers<16>(st, nblocks, t->row_ptr, M, XV, U, W, R, C, D, (double *)ctx->gslots.p); break;
            default: launch_helpers<32>(st, nblocks, t->row_ptr, M, XV, U, W, R, C, D, (double *)ctx->gslots.p); break;
        }
        double *Fsl = (double *)ctx->fslots.p;
        launch_fgemm(ctx, st, &b, J, U, row_slice, W, R, rps, (int)nsplit, Fsl);
    }
    const int64_t tot = (int64_t)J * R + R * R;
    if (ensure(ctx->fg, sizeof(double) * tot)) return DASH_E_CUDA;
    if (colsum(ctx, st, (double *)ctx->fslots.p, (M > 0 && N > 0) ? (int)nsplit : 0, (int64_t)J * R,
               (double *)ctx->fg.p) ||
        colsum(ctx, st, (double *)ctx->gslots.p, (M > 0 && N > 0) ? nblocks : 0, (int64_t)R * R,
               (double *)ctx->fg.p + (int64_t)J * R))
        return DASH_E_CUDA;
    k_finish_fg<<<(int)((tot + 255) / 256), 256, 0, st>>>((double *)ctx->fg.p, (double *)ctx->fsnap.p,
                                                           (double *)ctx->gsnap.p, 0.0, J, R, F, G);
    return cudaGetLastError() == cudaSuccess ? DASH_OK : DASH_E_CUDA;
}

}  // extern "C"

namespace {
// ---------------------------------------------------------------------------
// Row-parallel reconstruction error (local_error / slice_error and the ALS
// loss): per row e = sum_j phi(X[row][j] - sum_r z_r V[j][r]) with
// z = U[row] o W[state_row[slice(row)]] (local_error) or z = Z[row] (ALS:
// (Q H) o w already formed), phi = |.| or (.)^2.  One warp per row, lanes over
// the columns; V staged in shared memory (odd pitch) when it fits.  Then the
// per-slice sums in row order (one warp per slice) and a fixed-order tree
// over the slices: deterministic, and every X byte is read once at full
// occupancy (the previous one-warp-per-slice loops were latency-bound).
// ---------------------------------------------------------------------------
constexpr int kRecVS = 6144;  // J * R doubles staged (48 KB)
template <bool ABS, typename TX, typename TU>
__global__ void __launch_bounds__(256) k_row_err(const TX *__restrict__ X, int64_t ldx, int64_t N,
                                                 const TU *__restrict__ Z, int R, const double *__restrict__ V, int J,
                                                 const int32_t *__restrict__ row_slice,
                                                 const int32_t *__restrict__ state_row, const double *__restrict__ W,
                                                 double *__restrict__ row_err) {
    extern __shared__ double vs[];
    __shared__ double zbuf[8][DASH_MAX_RANK];
    const bool staged = (int64_t)J * R <= kRecVS;
    const int P = R + 1;
    if (staged)
        for (int i = threadIdx.x; i < J * R; i += blockDim.x) vs[(i / R) * P + i % R] = V[i];
    __syncthreads();
    const int lane = lane_id(), w = warp_id();
    double *zs = zbuf[w];
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + w, nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t row = gw; row < N; row += nw) {
        const double *wr = W ? W + (int64_t)state_row[row_slice[row]] * R : nullptr;
        for (int r = lane; r < R; r += 32) zs[r] = (double)Z[row * R + r] * (wr ? wr[r] : 1.0);
        __syncwarp();
        double acc = 0.0;
        for (int j = lane; j < J; j += 32) {
            double rec = 0.0;
            if (staged) {
                const double *vj = vs + j * P;
                for (int r = 0; r < R; ++r) rec = fma(zs[r], vj[r], rec);
            } else {
                const double *vj = V + (int64_t)j * R;
                for (int r = 0; r < R; ++r) rec = fma(zs[r], __ldg(vj + r), rec);
            }
            const double d = (double)X[row * ldx + j] - rec;
            acc = ABS ? acc + fabs(d) : fma(d, d, acc);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(FULL_MASK, acc, off);
        if (lane == 0) row_err[row] = acc;
        __syncwarp();
    }
}

// per-slice sum of the row errors (rows in order, lanes strided, fixed tree),
// divided by n_k * J when `mean` (local_error's per-slice mean)
__global__ void __launch_bounds__(256) k_seg_sum(const double *__restrict__ row_err,
                                                 const int64_t *__restrict__ row_ptr, int K, int J, int mean,
                                                 double *__restrict__ per) {
    const int lane = lane_id();
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (int k = gw; k < K; k += nw) {
        const int64_t r0 = row_ptr[k], r1 = row_ptr[k + 1];
        double acc = 0.0;
        for (int64_t i = r0 + lane; i < r1; i += 32) acc += row_err[i];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(FULL_MASK, acc, off);
        if (lane == 0) per[k] = mean ? acc / ((double)(r1 - r0) * J) : acc;
    }
}

// fixed-order sum (or mean) of n values by one block of 1,024 threads: strided partials in four
// independent chains per thread (a single dependent chain of 212 loads per thread took 91 us for
// the 54k slices of a large update), then a tree
constexpr int kTreeThreads = 1024;
__global__ void __launch_bounds__(kTreeThreads) k_tree_sum(const double *__restrict__ v, int n, int mean,
                                                           double *__restrict__ out) {
    __shared__ double part[kTreeThreads];
    double a4[4] = {0.0, 0.0, 0.0, 0.0};
    for (int i0 = threadIdx.x; i0 < n; i0 += 4 * kTreeThreads) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int i = i0 + q * kTreeThreads;
            if (i < n) a4[q] += v[i];
        }
    }
    part[threadIdx.x] = (a4[0] + a4[1]) + (a4[2] + a4[3]);
    __syncthreads();
    for (int h = kTreeThreads / 2; h > 0; h >>= 1) {
        if ((int)threadIdx.x < h) part[threadIdx.x] += part[threadIdx.x + h];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = mean ? (n > 0 ? part[0] / n : 0.0) : part[0];
}

// Same row errors with the reconstruction on the FP64 tensor cores: a warp takes 8 rows, its A
// fragments are the rows' Z (o w) values, B fragments come from V staged in shared memory (pitch
// RB + 4: the fragment's 8 x 4 reads hit distinct banks), one 8 x 8 tile of Z V^T per 8 columns;
// each lane then owns two reconstructed entries of one row, subtracts them from X and
// accumulates; the four lanes of a row are summed in a fixed order.  ~10x fewer instructions
// than the scalar loop above, which was shared-memory-issue bound at ~1 TB/s.
template <bool ABS, typename TX, typename TU, int RB>
__global__ void __launch_bounds__(256) k_row_err_mma(const TX *__restrict__ X, int64_t ldx, int64_t N,
                                                     const TU *__restrict__ Z, int R, const double *__restrict__ V,
                                                     int J, const int32_t *__restrict__ row_slice,
                                                     const int32_t *__restrict__ state_row,
                                                     const double *__restrict__ W, double *__restrict__ row_err) {
    constexpr int P = RB == 4 ? 4 : RB + 4, KS = RB / 4;
    extern __shared__ double vs[];  // J8 x P, zero padded
    const int J8 = (J + 7) / 8 * 8;
    for (int i = threadIdx.x; i < J8 * P; i += blockDim.x) {
        const int j = i / P, r = i % P;
        vs[i] = (j < J && r < R) ? V[(int64_t)j * R + r] : 0.0;
    }
    __syncthreads();
    const int lane = lane_id(), g = lane >> 2, t = lane & 3;
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id(), nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t nblk = (N + 7) / 8;
    for (int64_t blk = gw; blk < nblk; blk += nw) {
        const int64_t row = blk * 8 + g;
        const bool valid = row < N;
        const double *wr = (W && valid) ? W + (int64_t)state_row[row_slice[row]] * R : nullptr;
        double a[KS];
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
            const int r = 4 * kk + t;
            a[kk] = (valid && r < R) ? (double)Z[row * R + r] * (wr ? wr[r] : 1.0) : 0.0;
        }
        const TX *xrow = X + (valid ? row : 0) * ldx;
        double acc = 0.0;
#pragma unroll 4
        for (int j0 = 0; j0 < J8; j0 += 8) {
            const int j = j0 + 2 * t;
            const double x0 = (valid && j < J) ? (double)xrow[j] : 0.0;
            const double x1 = (valid && j + 1 < J) ? (double)xrow[j + 1] : 0.0;
            double c[2] = {0.0, 0.0};
            const double *vb = vs + (j0 + g) * P + t;
#pragma unroll
            for (int kk = 0; kk < KS; ++kk) dmma884(c, a[kk], vb[4 * kk]);
            const double d0 = x0 - c[0], d1 = x1 - c[1];  // padded columns: x = 0 and rec = 0
            acc = ABS ? acc + fabs(d0) + fabs(d1) : fma(d1, d1, fma(d0, d0, acc));
        }
        acc += __shfl_xor_sync(FULL_MASK, acc, 1);
        acc += __shfl_xor_sync(FULL_MASK, acc, 2);
        if (t == 0 && valid) row_err[row] = acc;
    }
}

// Wide-J form of k_row_err_mma (J x (RB + 4) doubles of V do not fit in shared memory: J = 1,024):
// a CTA takes 64 rows at a time (8 rows per warp, A fragments kept in registers) and walks the
// columns in chunks of JC, re-staging that chunk of V from L2 for every 64-row group (V traffic
// ~ X traffic).  The scalar fallback this replaces ran at 0.9 TB/s at R = 10 and 33 GB/s at R = 64.
template <bool ABS, typename TX, typename TU, int RB>
__global__ void __launch_bounds__(256) k_row_err_mma_wide(const TX *__restrict__ X, int64_t ldx, int64_t N,
                                                          const TU *__restrict__ Z, int R, const double *__restrict__ V,
                                                          int J, int JC, const int32_t *__restrict__ row_slice,
                                                          const int32_t *__restrict__ state_row,
                                                          const double *__restrict__ W, double *__restrict__ row_err) {
    constexpr int P = RB == 4 ? 4 : RB + 4, KS = RB / 4;
    extern __shared__ double vs[];  // JC x P
    const int lane = lane_id(), g = lane >> 2, t = lane & 3, w = warp_id();
    const int64_t ngroups = (N + 63) / 64;
    for (int64_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
        const int64_t row = grp * 64 + 8 * w + g;
        const bool valid = row < N;
        const double *wr = (W && valid) ? W + (int64_t)state_row[row_slice[row]] * R : nullptr;
        double a[KS];
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
            const int r = 4 * kk + t;
            a[kk] = (valid && r < R) ? (double)Z[row * R + r] * (wr ? wr[r] : 1.0) : 0.0;
        }
        const TX *xrow = X + (valid ? row : 0) * ldx;
        double acc = 0.0;
        for (int jc0 = 0; jc0 < J; jc0 += JC) {
            __syncthreads();  // the previous chunk (or group) is no longer read
            for (int i = threadIdx.x; i < JC * P; i += blockDim.x) {
                const int j = jc0 + i / P, r = i % P;
                vs[i] = (j < J && r < R) ? V[(int64_t)j * R + r] : 0.0;
            }
            __syncthreads();
            const int jn = min(JC, (J - jc0 + 7) / 8 * 8);
#pragma unroll 2
            for (int j0 = 0; j0 < jn; j0 += 8) {
                const int j = jc0 + j0 + 2 * t;
                const double x0 = (valid && j < J) ? (double)xrow[j] : 0.0;
                const double x1 = (valid && j + 1 < J) ? (double)xrow[j + 1] : 0.0;
                double c[2] = {0.0, 0.0};
                const double *vb = vs + (j0 + g) * P + t;
#pragma unroll
                for (int kk = 0; kk < KS; ++kk) dmma884(c, a[kk], vb[4 * kk]);
                const double d0 = x0 - c[0], d1 = x1 - c[1];
                acc = ABS ? acc + fabs(d0) + fabs(d1) : fma(d1, d1, fma(d0, d0, acc));
            }
        }
        acc += __shfl_xor_sync(FULL_MASK, acc, 1);
        acc += __shfl_xor_sync(FULL_MASK, acc, 2);
        if (t == 0 && valid) row_err[row] = acc;
    }
}

template <bool ABS, typename TX, typename TU, int RB>
void launch_row_err_mma_wide(dash_ctx *ctx, cudaStream_t st, const TX *X, int64_t ldx, int64_t N, const TU *Z, int R,
                             const double *V, int J, const int32_t *row_slice, const int32_t *state_row,
                             const double *W, double *row_err) {
    constexpr int P = RB == 4 ? 4 : RB + 4;
    const int JC = RB <= 16 ? 512 : (RB <= 32 ? 256 : 128);
    const size_t smem = sizeof(double) * (size_t)JC * P;
    ensure_smem_attr(k_row_err_mma_wide<ABS, TX, TU, RB>, smem);
    const int blocks = (int)std::min<int64_t>((N + 63) / 64, (int64_t)ctx->num_sms * 2);
    k_row_err_mma_wide<ABS, TX, TU, RB><<<std::max(blocks, 1), 256, smem, st>>>(X, ldx, N, Z, R, V, J, JC, row_slice,
                                                                                state_row, W, row_err);
}

template <bool ABS, typename TX, typename TU, int RB>
void launch_row_err_mma(dash_ctx *ctx, cudaStream_t st, const TX *X, int64_t ldx, int64_t N, const TU *Z, int R,
                        const double *V, int J, const int32_t *row_slice, const int32_t *state_row, const double *W,
                        double *row_err, size_t smem) {
    ensure_smem_attr(k_row_err_mma<ABS, TX, TU, RB>, smem);
    const int blocks = (int)std::min<int64_t>((N + 63) / 64, (int64_t)ctx->num_sms * 8);
    k_row_err_mma<ABS, TX, TU, RB><<<std::max(blocks, 1), 256, smem, st>>>(X, ldx, N, Z, R, V, J, row_slice,
                                                                           state_row, W, row_err);
}

template <bool ABS, typename TX, typename TU>
int launch_row_err(dash_ctx *ctx, cudaStream_t st, const TX *X, int64_t ldx, int64_t N, const TU *Z, int R,
                   const double *V, int J, const int32_t *row_slice, const int32_t *state_row, const double *W,
                   double *row_err) {
    if (N <= 0) return 0;
    {
        static const bool scalar = getenv("DASH_ROWERR_SCALAR") != nullptr;  // A/B switch
        const int RB = rank_bucket(R), P = RB == 4 ? 4 : RB + 4;
        const size_t sm = sizeof(double) * (size_t)((J + 7) / 8 * 8) * P;
        if (!scalar && sm > 96 * 1024) {  // wide J: V chunked through shared memory
            switch (RB) {
                case 4: launch_row_err_mma_wide<ABS, TX, TU, 4>(ctx, st, X, ldx, N, Z, R, V, J, row_slice, state_row, W, row_err); break;
                case 8: launch_row_err_mma_wide<ABS, TX, TU, 8>(ctx, st, X, ldx, N, Z, R, V, J, row_slice, state_row, W, row_err); break;
                case 16: launch_row_err_mma_wide<ABS, TX, TU, 16>(ctx, st, X, ldx, N, Z, R, V, J, row_slice, state_row, W, row_err); break;
                case 32: launch_row_err_mma_wide<ABS, TX, TU, 32>(ctx, st, X, ldx, N, Z, R, V, J, row_slice, state_row, W, row_err); break;
                default: launch_row_err_mma_wide<ABS, TX, TU, 64>(ctx, st, X, ldx, N, Z, R, V, J, row_slice, state_row, W, row_err); break;
            }
            return 0;
        }
        if (!scalar && sm <= 96 * 1024) {
            switch (RB) {
                case 4: launch_row_err_mma<ABS, TX, TU, 4>(ctx, st, X, ldx, N, Z, R, V, J, row_slice, state_row, W, row_err, sm); break;
                case 8: launch_row_err_mma<ABS, TX, TU, 8>(ctx, st, X, ldx, N, Z, R, V, J, row_slice, state_row, W, row_err, sm); break;
                case 16: launch_row_err_mma<ABS, TX, TU, 16>(ctx, st, X, ldx, N, Z, R, V, J, row_slice, state_row, W, row_err, sm); break;
                case 32: launch_row_err_mma<ABS, TX, TU, 32>(ctx, st, X, ldx, N, Z, R, V, J, row_slice, state_row, W, row_err, sm); break;
                default: launch_row_err_mma<ABS, TX, TU, 64>(ctx, st, X, ldx, N, Z, R, V, J, row_slice, state_row, W, row_err, sm); break;
            }
            return 0;
        }
    }
    const size_t smem = (int64_t)J * R <= kRecVS ? sizeof(double) * (size_t)J * (R + 1) : 0;
    ensure_smem_attr(k_row_err<ABS, TX, TU>, smem);
    const int blocks = (int)std::min<int64_t>((N + 7) / 8, (int64_t)ctx->num_sms * 8);
    k_row_err<ABS, TX, TU><<<std::max(blocks, 1), 256, smem, st>>>(X, ldx, N, Z, R, V, J, row_slice, state_row, W,
                                                                   row_err);
    return 0;
}

template <class B, typename TX>
int local_error_impl(dash_ctx *ctx, void *stream, const B *b, const TX *U, const double *W,
                         const double *V, int32_t J, int32_t R, double *slice_err, double *tensor_err) {
    if (!ctx || !b || R < 1 || R > DASH_MAX_RANK || J < 1) return DASH_E_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    const int M = b->M;
    const int64_t N = b->N;
    if (M > 0 && N > 0) {
        if (ensure(ctx->row_slice, sizeof(int32_t) * (size_t)N) || ensure(ctx->rerr, sizeof(double) * (size_t)N))
            return DASH_E_CUDA;
        k_row_slice<<<std::min(ctx->num_sms * 4, (M + 7) / 8 + 1), 256, 0, st>>>(b->row_ptr, M,
                                                                               (int32_t *)ctx->row_slice.p);
        launch_row_err<true>(ctx, st, b->X, b->ldx, N, U, R, V, J, (const int32_t *)ctx->row_slice.p, b->state_row,
                             W, (double *)ctx->rerr.p);
        k_seg_sum<<<std::max(1, std::min((M + 7) / 8, ctx->num_sms * 8)), 256, 0, st>>>(
            (const double *)ctx->rerr.p, b->row_ptr, M, J, 1, slice_err);
    }
    k_tree_sum<<<1, kTreeThreads, 0, st>>>(slice_err, M, 1, tensor_err);
    return cudaGetLastError() == cudaSuccess ? DASH_OK : DASH_E_CUDA;
}

}  // namespace

extern "C" {

int dash_local_error_f64(dash_ctx *ctx, void *stream, const dash_batch_f64 *b, const double *U, const double *W,
                         const double *V, int32_t J, int32_t R, double *slice_err, double *tensor_err) {
    return local_error_impl(ctx, stream, b, U, W, V, J, R, slice_err, tensor_err);
}

int dash_local_error_f32(dash_ctx *ctx, void *stream, const dash_batch_f32 *b, const float *U, const double *W,
                         const double *V, int32_t J, int32_t R, double *slice_err, double *tensor_err) {
    return local_error_impl(ctx, stream, b, U, W, V, J, R, slice_err, tensor_err);
}

int dash_ridge_solve_f64(dash_ctx *ctx, void *stream, int32_t B, int32_t n, int32_t m, const double *lhs,
                         const double *rhs, double *x, double eps) {
    if (!ctx || B < 0 || n < 1 || n > DASH_MAX_RANK_ALS || m < 0) return DASH_E_ARG;
    if (B == 0 || m == 0) return DASH_OK;
    cudaStream_t st = (cudaStream_t)stream;
    switch (rank_bucket(n)) {
        case 4: launch_ridge<4>(st, B, lhs, rhs, n, m, eps, x, ctx->err); break;
        case 8: launch_ridge<8>(st, B, lhs, rhs, n, m, eps, x, ctx->err); break;
        case 16: launch_ridge<16>(st, B, lhs, rhs, n, m, eps, x, ctx->err); break;
        default: launch_ridge<32>(st, B, lhs, rhs, n, m, eps, x, ctx->err); break;
    }
    return cudaGetLastError() == cudaSuccess ? DASH_OK : DASH_E_CUDA;
}

}  // extern "C"
