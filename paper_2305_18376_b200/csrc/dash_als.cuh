// Static PARAFAC2-ALS sweep on the GPU -- the fit behind initialize()
// (als.py:102-201 of the reference).  One sweep = dash_als_sweep_f64:
//
//   k_xv          XV = X V                                   (DMMA, shared with the update)
//   k_als_polar   per slice: T = (XV o w_k) H^T, Q_k = polar(T) (als.py:155-164),
//                 yv_k = Q_k^T X_k V = Q_k^T XV_k (the (K,R,R) projected tensor times V,
//                 als.py:168).  polar() = CholQR2 (T = Q2 R2 R1) + one-sided Jacobi
//                 SVD of the R x R factor: error ~ eps*cond(T), like LAPACK gesdd,
//                 instead of the Gram route's eps*cond(T)^2.
//   k_als_cp      H, W solves of the CP sweep (als.py:166-176), one CTA
//   k_als_qh      Z = (Q_k H) o w_k per row
//   k_fgemm       rhs_v = X^T Z  (= einsum('krj,rz,kz->jz', Y, H, W), als.py:177)
//   k_ridge       V = ridge_solve(hth o wtw, rhs_v^T)^T        (als.py:178)
//   k_als_loss    sum_k ||X_k - Z_k V^T||^2, direct form        (als.py:182-185)
#pragma once

namespace {

// Forward substitution only: solve L y = b (lane-held b, L in shared memory).
template <int RB>
__device__ __forceinline__ void fwd_solve_lane(const double *L, int ld, const double *dinv, double (&b)[RB]) {
#pragma unroll
    for (int k = 0; k < RB; ++k) {
        b[k] *= lds_nohoist(dinv + k);
#pragma unroll
        for (int i = k + 1; i < RB; ++i) b[i] = fma(-lds_nohoist(L + i * ld + k), b[k], b[i]);
    }
}

// Accumulate gram pairs sum_i rows[i][a] * rows[i][c] over 32 staged rows.
template <int NPL>
__device__ __forceinline__ void pair_accum(const double *A, const double *B, int ld, const int *pa, const int *pc,
                                           int npairs, double (&acc)[NPL]) {
    const int lane = lane_id();
#pragma unroll
    for (int q = 0; q < NPL; ++q) {
        const int pp = lane + 32 * q;
        if (pp < npairs) {
            const int a = pa[pp], c = pc[pp];
            double s = acc[q];
            for (int i = 0; i < 32; ++i) s = fma(A[i * ld + a], B[i * ld + c], s);
            acc[q] = s;
        }
    }
}

template <int RB>
struct AlsSmem {
    static constexpr int LD = RB + 1;
    // per warp: rows[32*LD], rows2[32*LD], L1[RB*LD], L2[RB*LD], M[RB*LD], S[RB*LD], d1[RB], d2[RB], w[RB]
    static constexpr int per_warp = 2 * 32 * LD + 4 * RB * LD + 3 * RB;
    static constexpr int NP = RB * (RB + 1) / 2;
    static constexpr int NQ = RB * RB;
    // shared: H[RB*LD] + pair tables (NP + NQ) * 2 ints
    static constexpr int shared = RB * LD + (NP + NQ);
    __host__ __device__ static constexpr size_t bytes(int nw) { return sizeof(double) * (shared + nw * per_warp); }
};

template <int RB, int NW>
__global__ void __launch_bounds__(NW * 32) k_als_polar(const int64_t *__restrict__ row_ptr, int K,
                                                       const double *__restrict__ XV, const double *__restrict__ W,
                                                       const double *__restrict__ H, int R, double *__restrict__ T,
                                                       double *__restrict__ Q, double *__restrict__ yv,
                                                       unsigned long long *err) {
    using S = AlsSmem<RB>;
    constexpr int LD = S::LD, NP = S::NP, NQ = S::NQ;
    constexpr int NPL = (NP + 31) / 32, NQL = (NQ + 31) / 32;
    extern __shared__ double sm[];
    double *Hs = sm;
    int *pa = reinterpret_cast<int *>(Hs + RB * LD);  // NP sym pairs then NQ full pairs
    int *pc = pa + NP + NQ;
    const int lane = lane_id(), w = warp_id();
    double *base = sm + S::shared + w * S::per_warp;
    double *rows = base, *rows2 = rows + 32 * LD;
    double *L1 = rows2 + 32 * LD, *L2 = L1 + RB * LD, *Ms = L2 + RB * LD, *Ss = Ms + RB * LD;
    double *d1 = Ss + RB * LD, *d2 = d1 + RB, *wv = d2 + RB;
    for (int i = threadIdx.x; i < RB * LD; i += blockDim.x) {
        int r = i / LD, z = i % LD;
        Hs[i] = (r < R && z < R) ? H[r * R + z] : 0.0;
    }
    for (int i = threadIdx.x; i < NP + NQ; i += blockDim.x) {
        int r, z;
        if (i < NP) {
            pair_rz(i, RB, r, z);
        } else {
            r = (i - NP) / RB;
            z = (i - NP) % RB;
        }
        pa[i] = r;
        pc[i] = z;
    }
    __syncthreads();
    // one warp per slice.  (One CTA per slice with the warps sharing its chunks was measured
    // slower -- 3.99 -> 5.05 ms at the daily shape: the kernel is bound by its scalar row passes,
    // not by its longest slice, and the redundant per-warp factorisations cost SM time.)
    const int gw = blockIdx.x * NW + w, nwarps = gridDim.x * NW;
    for (int k = gw; k < K; k += nwarps) {
        const int64_t r0 = row_ptr[k], r1 = row_ptr[k + 1];
        if (lane < RB) wv[lane] = lane < R ? W[(int64_t)k * R + lane] : 0.0;
        __syncwarp();
        // ---- pass 1: T rows (als.py:156) and S1 = T^T T
        double g1[NPL];
#pragma unroll
        for (int q = 0; q < NPL; ++q) g1[q] = 0.0;
        for (int64_t c0 = r0; c0 < r1; c0 += 32) {
            const int64_t row = c0 + lane;
            const bool valid = row < r1;
            double xw[RB];
#pragma unroll
            for (int z = 0; z < RB; ++z) xw[z] = (valid && z < R) ? XV[row * R + z] * wv[z] : 0.0;
#pragma unroll
            for (int r = 0; r < RB; ++r) {
                double t = 0.0;
#pragma unroll
                for (int z = 0; z < RB; ++z) t = fma(xw[z], Hs[r * LD + z], t);
                rows[lane * LD + r] = t;
                if (valid && r < R) T[row * R + r] = t;
            }
            __syncwarp();
            pair_accum<NPL>(rows, rows, LD, pa, pc, NP, g1);
            __syncwarp();
        }
        // ---- S1 -> L1 (S1 = L1 L1^T, R1 = L1^T)
#pragma unroll
        for (int q = 0; q < NPL; ++q) {
            const int pp = lane + 32 * q;
            if (pp < NP) {
                Ss[pa[pp] * LD + pc[pp]] = g1[q];
                Ss[pc[pp] * LD + pa[pp]] = g1[q];
            }
        }
        __syncwarp();
        bool ok;
        {
            double rr[RB];
#pragma unroll
            for (int z = 0; z < RB; ++z) rr[z] = (lane < R && z < R) ? Ss[lane * LD + z] : (lane == z ? 1.0 : 0.0);
            ok = chol_regs<RB>(rr, L1, LD, d1);
        }
        // ---- pass 2: Q1 = T L1^-T (in place in T) and S2 = Q1^T Q1
        double g2[NPL];
#pragma unroll
        for (int q = 0; q < NPL; ++q) g2[q] = 0.0;
        for (int64_t c0 = r0; c0 < r1; c0 += 32) {
            const int64_t row = c0 + lane;
            const bool valid = row < r1;
            double b[RB];
#pragma unroll
            for (int r = 0; r < RB; ++r) b[r] = (valid && r < R) ? T[row * R + r] : 0.0;
            fwd_solve_lane<RB>(L1, LD, d1, b);
#pragma unroll
            for (int r = 0; r < RB; ++r) {
                if (!valid) b[r] = 0.0;
                rows[lane * LD + r] = b[r];
                if (valid && r < R) T[row * R + r] = b[r];
            }
            __syncwarp();
            pair_accum<NPL>(rows, rows, LD, pa, pc, NP, g2);
            __syncwarp();
        }
#pragma unroll
        for (int q = 0; q < NPL; ++q) {
            const int pp = lane + 32 * q;
            if (pp < NP) {
                Ss[pa[pp] * LD + pc[pp]] = g2[q];
                Ss[pc[pp] * LD + pa[pp]] = g2[q];
            }
        }
        __syncwarp();
        {
            double rr[RB];
#pragma unroll
            for (int z = 0; z < RB; ++z) rr[z] = (lane < R && z < R) ? Ss[lane * LD + z] : (lane == z ? 1.0 : 0.0);
            ok = chol_regs<RB>(rr, L2, LD, d2) && ok;
        }
        if (!ok && lane == 0) report_error(err, k, DASH_E_SINGULAR);
        // ---- Rt = R2 R1 = L2^T L1^T into Ms (row i by lane i); Va = I into Ss
        double *Rt = Ms, *Va = Ss;
        if (lane < RB) {
            for (int j = 0; j < RB; ++j) {
                double acc = 0.0;
                for (int m = 0; m < RB; ++m) acc = fma(L2[m * LD + lane], L1[j * LD + m], acc);
                Rt[lane * LD + j] = acc;
                Va[lane * LD + j] = (lane == j) ? 1.0 : 0.0;
            }
        }
        __syncwarp();
        // ---- one-sided Jacobi SVD of Rt (cyclic by rows): Rt V = U Sigma
        for (int sweep = 0; sweep < 60; ++sweep) {
            double offmax = 0.0;
            for (int p = 0; p < R - 1; ++p) {
                for (int q = p + 1; q < R; ++q) {
                    const double a = lane < RB ? Rt[lane * LD + p] : 0.0;
                    const double b = lane < RB ? Rt[lane * LD + q] : 0.0;
                    double al = a * a, be = b * b, ga = a * b;
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) {
                        al += __shfl_xor_sync(FULL_MASK, al, off);
                        be += __shfl_xor_sync(FULL_MASK, be, off);
                        ga += __shfl_xor_sync(FULL_MASK, ga, off);
                    }
                    const double nrm = sqrt(al * be);
                    if (!(nrm > 0.0) || fabs(ga) <= 1e-16 * nrm) continue;  // warp-uniform
                    offmax = fmax(offmax, fabs(ga) / nrm);
                    const double zeta = (be - al) / (2.0 * ga);
                    const double tt = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                    const double cs = 1.0 / sqrt(1.0 + tt * tt), sn = cs * tt;
                    if (lane < RB) {
                        Rt[lane * LD + p] = cs * a - sn * b;
                        Rt[lane * LD + q] = sn * a + cs * b;
                        const double vp = Va[lane * LD + p], vq = Va[lane * LD + q];
                        Va[lane * LD + p] = cs * vp - sn * vq;
                        Va[lane * LD + q] = sn * vp + cs * vq;
                    }
                    __syncwarp();
                }
            }
            if (offmax <= 1e-15) break;
        }
        // ---- polar(Rt) = U V^T with U = Rt V Sigma^-1 (columns of the rotated Rt
        // normalised); P row i = sum_m U[i][m] V[j][m].  Then M = L2^-T P so that
        // Q = Q1 M = Q2 polar(Rt) = polar(T).
        {
            double sig[RB];
#pragma unroll
            for (int m = 0; m < RB; ++m) {
                const double v = lane < RB ? Rt[lane * LD + m] : 0.0;
                sig[m] = v * v;
            }
            warp_allreduce<RB>(sig);
#pragma unroll
            for (int m = 0; m < RB; ++m) sig[m] = (m < R && sig[m] > 0.0) ? 1.0 / sqrt(sig[m]) : 0.0;
            double prow[RB];
#pragma unroll
            for (int j = 0; j < RB; ++j) {
                double acc = 0.0;
                if (lane < RB) {
#pragma unroll
                    for (int m = 0; m < RB; ++m) acc = fma(Rt[lane * LD + m] * sig[m], Va[j * LD + m], acc);
                }
                prow[j] = (j < R && lane < R) ? acc : (j == lane ? 1.0 : 0.0);
            }
            __syncwarp();
            // M = L2^-T P: column c of M solves L2^T m = p_c; do it lane-per-column
            if (lane < RB) {
#pragma unroll
                for (int j = 0; j < RB; ++j) Rt[lane * LD + j] = prow[j];  // Rt <- P (row-major)
            }
            __syncwarp();
            double col[RB];
#pragma unroll
            for (int i = 0; i < RB; ++i) col[i] = lane < RB ? Rt[i * LD + lane] : 0.0;
#pragma unroll
            for (int kk = RB - 1; kk >= 0; --kk) {
                col[kk] *= d2[kk];
#pragma unroll
                for (int i = 0; i < kk; ++i) col[i] = fma(-L2[kk * LD + i], col[kk], col[i]);
            }
            __syncwarp();
            if (lane < RB) {
#pragma unroll
                for (int i = 0; i < RB; ++i) Va[i * LD + lane] = col[i];  // Va <- M
            }
            __syncwarp();
        }
        // ---- pass 3: Q = Q1 M (output) and yv = Q^T XV (full R x R)
        double gy[NQL];
#pragma unroll
        for (int q = 0; q < NQL; ++q) gy[q] = 0.0;
        for (int64_t c0 = r0; c0 < r1; c0 += 32) {
            const int64_t row = c0 + lane;
            const bool valid = row < r1;
            double q1[RB];
#pragma unroll
            for (int r = 0; r < RB; ++r) q1[r] = (valid && r < R) ? T[row * R + r] : 0.0;
#pragma unroll
            for (int j = 0; j < RB; ++j) {
                double acc = 0.0;
#pragma unroll
                for (int i = 0; i < RB; ++i) acc = fma(q1[i], Va[i * LD + j], acc);
                if (!valid || j >= R) acc = 0.0;
                rows[lane * LD + j] = acc;
                rows2[lane * LD + j] = (valid && j < R) ? XV[row * R + j] : 0.0;
                if (valid && j < R) Q[row * R + j] = acc;
            }
            __syncwarp();
            pair_accum<NQL>(rows, rows2, LD, pa + NP, pc + NP, NQ, gy);
            __syncwarp();
        }
#pragma unroll
        for (int q = 0; q < NQL; ++q) {
            const int pp = lane + 32 * q;
            if (pp < NQ) {
                const int r = pa[NP + pp], z = pc[NP + pp];
                if (r < R && z < R) yv[(int64_t)k * R * R + r * R + z] = gy[q];
            }
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// k_als_polar_mma: the same per-slice polar factor (CholQR2 + Jacobi, als.py:156-160)
// with the three row passes on the FP64 tensor cores.  Each pass is
//     out (8 x RB) = in (8 x RB) . B (RB x RB)   per 8-row chunk,
// followed by a Gram accumulation of the chunk:
//   pass 1: in = XV o w,  B = H^T       -> T,   S1 += T^T T
//   pass 2: in = T,       B = L1^{-T}   -> Q1 (in place), S2 += Q1^T Q1
//   pass 3: in = Q1,      B = M         -> Q,   yv += Q^T XV
// (L1^{-1} is formed explicitly, lane per column, instead of a forward
// substitution per row; CholQR2's second pass absorbs the difference.)  Chunks
// live in shared memory as swizzled 8 x 8 tiles (swk::toff), so the A / B /
// transposed DMMA fragment patterns of dash_slicesw.cuh apply unchanged.  The
// scalar kernel above spent ~600 FMA + as many LDS per row; this one ~14 DMMA
// per 8 rows and pass.  One warp per slice; the R x R serial part (Cholesky
// twice, the Jacobi SVD, M) is the scalar kernel's.
// ---------------------------------------------------------------------------
template <int NB>
struct AlsMmaSmem {
    static constexpr int RB = 8 * NB, LD = RB + 1;
    // per warp: In[NB] | Out[NB] | Xt[NB] | Bm[NB*NB] tiles, L1, L2, Ms, Ss (RB x LD), d1, d2, wv
    static constexpr int per_warp = (3 * NB + NB * NB) * 64 + 4 * RB * LD + 3 * RB;
    static constexpr int shared = NB * NB * 64;  // H^T tiles
    static constexpr int NRL = NB * NB * 2;      // Gram values per lane (the full yv block is the largest)
    // + red[nw][NRL * 32]: per-warp Gram partials of the cooperative variant
    __host__ __device__ static constexpr size_t bytes(int nw, bool coop) {
        return sizeof(double) * (shared + nw * per_warp + (coop ? nw * NRL * 32 : 0));
    }
};

// COOP = false: one warp per slice of `list` (short slices).  COOP = true: one CTA per slice -- its
// warps take the slice's chunks in turn and add their Gram partials in warp order through shared
// memory (long slices: a 4,000-row slice is 1,500 serial chunk passes for a single warp); the R x R
// serial part is then repeated by every warp on identical inputs.
template <int NB, int NW, bool COOP>
__global__ void __launch_bounds__(NW * 32, NB == 2 ? 3 : 1) k_als_polar_mma(const int64_t *__restrict__ row_ptr,
                                                           const int32_t *__restrict__ list, int K,
                                                           const double *__restrict__ XV, const double *__restrict__ W,
                                                           const double *__restrict__ H, int R, double *__restrict__ T,
                                                           double *__restrict__ Q, double *__restrict__ yv,
                                                           unsigned long long *err) {
    using namespace swk;
    using S = AlsMmaSmem<NB>;
    constexpr int RB = S::RB, LD = S::LD, NT = NB * (NB + 1) / 2;
    extern __shared__ double sm[];
    double *BH = sm;  // tile (kb, jb) element (k, n) = H[8 jb + n][8 kb + k]
    const int lane = lane_id(), w = warp_id();
    double *base = sm + S::shared + w * S::per_warp;
    double *In = base, *Out = In + NB * 64, *Xt = Out + NB * 64, *Bm = Xt + NB * 64;
    double *L1 = Bm + NB * NB * 64, *L2 = L1 + RB * LD, *Ms = L2 + RB * LD, *Ss = Ms + RB * LD;
    double *d1 = Ss + RB * LD, *d2 = d1 + RB, *wv = d2 + RB;
    for (int i = threadIdx.x; i < NB * NB * 64; i += blockDim.x) {
        const int tl = i >> 6, e = i & 63, kb = tl / NB, jb = tl % NB;
        const int k = e >> 3, n = (e & 7) ^ ((k & 2) << 1);  // inverse of toff(k, n) = 8 k + (n ^ ...)
        const int hr = 8 * jb + n, hc = 8 * kb + k;
        BH[i] = (hr < R && hc < R) ? H[hr * R + hc] : 0.0;
    }
    __syncthreads();
    const LaneOff o = lane_offsets();
    const int g = o.g, c0 = o.c0;
    double *red = sm + S::shared + NW * S::per_warp;
    // cooperative variant: Gram partials of the CTA's warps -> the full sum in every warp (warp order)
    auto reduce = [&](auto &acc) {
        if constexpr (COOP) {
            constexpr int n = (int)(sizeof(acc) / sizeof(double));
            double *flat = &acc[0][0];
#pragma unroll
            for (int q = 0; q < n; ++q) red[(w * S::NRL + q) * 32 + lane] = flat[q];
            __syncthreads();
#pragma unroll
            for (int q = 0; q < n; ++q) {
                double t = 0.0;
                for (int ww = 0; ww < NW; ++ww) t += red[(ww * S::NRL + q) * 32 + lane];
                flat[q] = t;
            }
            __syncthreads();
        }
    };
    const int cw = COOP ? w : 0, cs = COOP ? NW : 1;  // this warp's first chunk and the chunk stride
    // out tiles (C layout, registers) = In . B, B given as NB x NB tiles
    auto gemm = [&](const double *Bt, double (&out)[NB][2]) {
#pragma unroll
        for (int jb = 0; jb < NB; ++jb) {
            out[jb][0] = out[jb][1] = 0.0;
#pragma unroll
            for (int kb = 0; kb < NB; ++kb) mma_xy(out[jb], In + 64 * kb, Bt + 64 * (kb * NB + jb), o);
        }
    };
    // rows of a chunk (global, R columns) -> registers (optionally scaled by wv) -> tiles; the next
    // chunk is fetched before the current one is worked on, so its latency hides behind the DMMAs
    auto fetch = [&](double (&v)[NB][2], const double *src, int64_t row, bool valid, bool scale) {
#pragma unroll
        for (int kb = 0; kb < NB; ++kb)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int col = 8 * kb + c0 + e;
                double x = (valid && col < R) ? src[row * R + col] : 0.0;
                if (scale) x *= wv[col];
                v[kb][e] = x;
            }
    };
    auto put = [&](double *Tl, const double (&v)[NB][2]) {
#pragma unroll
        for (int kb = 0; kb < NB; ++kb) stc(Tl + 64 * kb, v[kb], o);
    };
    auto copy2 = [&](double (&d)[NB][2], const double (&a)[NB][2]) {
#pragma unroll
        for (int kb = 0; kb < NB; ++kb) d[kb][0] = a[kb][0], d[kb][1] = a[kb][1];
    };
    auto store_rows = [&](double *dst, int64_t row, bool valid, const double (&out)[NB][2]) {
#pragma unroll
        for (int jb = 0; jb < NB; ++jb) {
            stc(Out + 64 * jb, out[jb], o);
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int col = 8 * jb + c0 + e;
                if (valid && col < R) dst[row * R + col] = out[jb][e];
            }
        }
    };
    // symmetric Gram tiles -> the lower triangle of Ss (row-major)
    auto gram_to_ss = [&](const double (&ga)[NT][2]) {
#pragma unroll
        for (int ib = 0; ib < NB; ++ib)
#pragma unroll
            for (int kb = 0; kb <= ib; ++kb)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int r = 8 * ib + g, c = 8 * kb + c0 + e;
                    if (ib > kb || r >= c) Ss[r * LD + c] = ga[tri(ib, kb)][e];  // lower triangle only (one writer each)
                }
    };
    const int gw = COOP ? blockIdx.x : blockIdx.x * NW + w, nwarps = COOP ? gridDim.x : gridDim.x * NW;
    for (int ki = gw; ki < K; ki += nwarps) {
        const int k = list[ki];
        const int64_t r0 = row_ptr[k], r1 = row_ptr[k + 1];
        const int nch = (int)((r1 - r0 + 7) >> 3);
        __syncwarp();
        for (int r = lane; r < RB; r += 32) wv[r] = r < R ? W[(int64_t)k * R + r] : 0.0;
        __syncwarp();
        // ---- pass 1
        double ga[NT][2];
#pragma unroll
        for (int t = 0; t < NT; ++t) ga[t][0] = ga[t][1] = 0.0;
        double cur[NB][2], nxt[NB][2];
        fetch(cur, XV, r0 + 8 * (int64_t)cw + g, r0 + 8 * (int64_t)cw + g < r1, true);
        for (int ch = cw; ch < nch; ch += cs) {
            const int64_t row = r0 + 8 * (int64_t)ch + g;
            const bool valid = row < r1;
            fetch(nxt, XV, row + 8 * cs, row + 8 * cs < r1, true);
            put(In, cur);
            __syncwarp();
            double out[NB][2];
            gemm(BH, out);
            store_rows(T, row, valid, out);
            __syncwarp();
#pragma unroll
            for (int ib = 0; ib < NB; ++ib)
#pragma unroll
                for (int kb = 0; kb <= ib; ++kb) mma_xty(ga[tri(ib, kb)], Out + 64 * ib, Out + 64 * kb, o);
            __syncwarp();
            copy2(cur, nxt);  // only now: the fetch had the whole chunk to land
        }
        reduce(ga);
        gram_to_ss(ga);
        __syncwarp();
        bool ok;
        {
            double rr[RB];
#pragma unroll
            for (int z = 0; z < RB; ++z)
                rr[z] = (lane < R && z < R) ? Ss[(lane >= z ? lane : z) * LD + (lane >= z ? z : lane)]
                                            : (lane == z ? 1.0 : 0.0);
            ok = chol_regs<RB>(rr, L1, LD, d1);
        }
        // ---- B = L1^{-T}: lane c solves L1 x = e_c; Bm (k = c, n = i) = x[i]
        {
            double x[RB];
#pragma unroll
            for (int i = 0; i < RB; ++i) x[i] = (i == lane) ? 1.0 : 0.0;
            if (lane < RB) fwd_solve_lane<RB>(L1, LD, d1, x);
            if (lane < RB) {
#pragma unroll
                for (int i = 0; i < RB; ++i) Bm[64 * ((lane >> 3) * NB + (i >> 3)) + toff(lane & 7, i & 7)] = x[i];
            }
        }
        __syncwarp();
        // ---- pass 2
#pragma unroll
        for (int t = 0; t < NT; ++t) ga[t][0] = ga[t][1] = 0.0;
        fetch(cur, T, r0 + 8 * (int64_t)cw + g, r0 + 8 * (int64_t)cw + g < r1, false);
        for (int ch = cw; ch < nch; ch += cs) {
            const int64_t row = r0 + 8 * (int64_t)ch + g;
            const bool valid = row < r1;
            fetch(nxt, T, row + 8 * cs, row + 8 * cs < r1, false);
            put(In, cur);
            __syncwarp();
            double out[NB][2];
            gemm(Bm, out);
            store_rows(T, row, valid, out);
            __syncwarp();
#pragma unroll
            for (int ib = 0; ib < NB; ++ib)
#pragma unroll
                for (int kb = 0; kb <= ib; ++kb) mma_xty(ga[tri(ib, kb)], Out + 64 * ib, Out + 64 * kb, o);
            __syncwarp();
            copy2(cur, nxt);  // only now: the fetch had the whole chunk to land
        }
        reduce(ga);
        gram_to_ss(ga);
        __syncwarp();
        {
            double rr[RB];
#pragma unroll
            for (int z = 0; z < RB; ++z)
                rr[z] = (lane < R && z < R) ? Ss[(lane >= z ? lane : z) * LD + (lane >= z ? z : lane)]
                                            : (lane == z ? 1.0 : 0.0);
            ok = chol_regs<RB>(rr, L2, LD, d2) && ok;
        }
        if (!ok && lane == 0 && cw == 0) report_error(err, k, DASH_E_SINGULAR);
        // ---- Rt = L2^T L1^T into Ms (row i by lane i); Va = I into Ss
        double *Rt = Ms, *Va = Ss;
        if (lane < RB) {
            for (int j = 0; j < RB; ++j) {
                double acc = 0.0;
                for (int m = 0; m < RB; ++m) acc = fma(L2[m * LD + lane], L1[j * LD + m], acc);
                Rt[lane * LD + j] = acc;
                Va[lane * LD + j] = (lane == j) ? 1.0 : 0.0;
            }
        }
        __syncwarp();
        // ---- one-sided Jacobi SVD of Rt (cyclic by rows): Rt V = U Sigma.  Column norms are
        // refreshed once per sweep (one batched warp reduction) and updated in closed form after
        // each rotation (|a'|^2 = |a|^2 - t gamma, |b'|^2 = |b|^2 + t gamma), so a pair costs one
        // warp reduction (gamma) instead of three; the rotation parameters come from rsqrt / rcp
        // seeds + Newton steps instead of three IEEE sqrt and three divisions (together 46% of the
        // kernel's stall samples at the daily shape, profiles/r02s3_als/ncu_polar_lines.txt).
        double *nrm2 = wv;  // the slice's weights are dead after pass 1
        for (int sweep = 0; sweep < 60; ++sweep) {
            {
                double sig[RB];
#pragma unroll
                for (int m = 0; m < RB; ++m) {
                    const double v = lane < RB ? Rt[lane * LD + m] : 0.0;
                    sig[m] = v * v;
                }
                warp_allreduce<RB>(sig);
                __syncwarp();
#pragma unroll
                for (int m = 0; m < RB; ++m)
                    if (lane == 0) nrm2[m] = sig[m];
                __syncwarp();
            }
            // (A round-robin ordering -- n / 2 independent rotations per round, batched reductions
            // -- was measured slower: 168 -> 255 registers, 2 CTAs per SM; polar 2.20 -> 2.66 ms daily.)
            double offmax = 0.0;
            for (int p = 0; p < R - 1; ++p) {
                for (int q = p + 1; q < R; ++q) {
                    const double a = lane < RB ? Rt[lane * LD + p] : 0.0;
                    const double b = lane < RB ? Rt[lane * LD + q] : 0.0;
                    const double al = nrm2[p], be = nrm2[q];
                    double gm = a * b;
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) gm += __shfl_xor_sync(FULL_MASK, gm, off);
                    const double ab = al * be;
                    if (!(ab > 0.0)) continue;                            // warp-uniform
                    const double rel = fabs(gm) * rsqrt_nr(ab);           // |gamma| / (|a| |b|)
                    if (rel <= 1e-16) continue;
                    offmax = fmax(offmax, rel);
                    const double zeta = (be - al) * 0.5 * rcp_nr(gm);
                    const double z1 = 1.0 + zeta * zeta;
                    const double tt = copysign(1.0, zeta) * rcp_nr(fabs(zeta) + z1 * rsqrt_nr(z1));
                    const double cs = rsqrt_nr(1.0 + tt * tt), sn = cs * tt;
                    if (lane < RB) {
                        Rt[lane * LD + p] = cs * a - sn * b;
                        Rt[lane * LD + q] = sn * a + cs * b;
                        const double vp = Va[lane * LD + p], vq = Va[lane * LD + q];
                        Va[lane * LD + p] = cs * vp - sn * vq;
                        Va[lane * LD + q] = sn * vp + cs * vq;
                    }
                    if (lane == 0) {
                        nrm2[p] = al - tt * gm;
                        nrm2[q] = be + tt * gm;
                    }
                    __syncwarp();
                }
            }
            if (offmax <= 1e-15) break;
        }
        // ---- polar(Rt) = U V^T, M = L2^-T polar(Rt); Bm (k = i, n = lane) = M[i][lane]
        {
            double sig[RB];
#pragma unroll
            for (int m = 0; m < RB; ++m) {
                const double v = lane < RB ? Rt[lane * LD + m] : 0.0;
                sig[m] = v * v;
            }
            warp_allreduce<RB>(sig);
#pragma unroll
            for (int m = 0; m < RB; ++m) sig[m] = (m < R && sig[m] > 0.0) ? 1.0 / sqrt(sig[m]) : 0.0;
            double prow[RB];
#pragma unroll
            for (int j = 0; j < RB; ++j) {
                double acc = 0.0;
                if (lane < RB) {
#pragma unroll
                    for (int m = 0; m < RB; ++m) acc = fma(Rt[lane * LD + m] * sig[m], Va[j * LD + m], acc);
                }
                prow[j] = (j < R && lane < R) ? acc : (j == lane ? 1.0 : 0.0);
            }
            __syncwarp();
            if (lane < RB) {
#pragma unroll
                for (int j = 0; j < RB; ++j) Rt[lane * LD + j] = prow[j];  // Rt <- P (row-major)
            }
            __syncwarp();
            double col[RB];
#pragma unroll
            for (int i = 0; i < RB; ++i) col[i] = lane < RB ? Rt[i * LD + lane] : 0.0;
#pragma unroll
            for (int kk = RB - 1; kk >= 0; --kk) {
                col[kk] *= d2[kk];
#pragma unroll
                for (int i = 0; i < kk; ++i) col[i] = fma(-L2[kk * LD + i], col[kk], col[i]);
            }
            __syncwarp();
            if (lane < RB) {
#pragma unroll
                for (int i = 0; i < RB; ++i) Bm[64 * ((i >> 3) * NB + (lane >> 3)) + toff(i & 7, lane & 7)] = col[i];
            }
            __syncwarp();
        }
        // ---- pass 3: Q = Q1 M, yv = Q^T XV (full RB x RB)
        double gy[NB * NB][2];
#pragma unroll
        for (int t = 0; t < NB * NB; ++t) gy[t][0] = gy[t][1] = 0.0;
        double curx[NB][2], nxtx[NB][2];
        fetch(cur, T, r0 + 8 * (int64_t)cw + g, r0 + 8 * (int64_t)cw + g < r1, false);
        fetch(curx, XV, r0 + 8 * (int64_t)cw + g, r0 + 8 * (int64_t)cw + g < r1, false);
        for (int ch = cw; ch < nch; ch += cs) {
            const int64_t row = r0 + 8 * (int64_t)ch + g;
            const bool valid = row < r1;
            fetch(nxt, T, row + 8 * cs, row + 8 * cs < r1, false);
            fetch(nxtx, XV, row + 8 * cs, row + 8 * cs < r1, false);
            put(In, cur);
            put(Xt, curx);
            __syncwarp();
            double out[NB][2];
            gemm(Bm, out);
            store_rows(Q, row, valid, out);
            __syncwarp();
#pragma unroll
            for (int ib = 0; ib < NB; ++ib)
#pragma unroll
                for (int kb = 0; kb < NB; ++kb) mma_xty(gy[ib * NB + kb], Out + 64 * ib, Xt + 64 * kb, o);
            __syncwarp();
            copy2(cur, nxt);
            copy2(curx, nxtx);
        }
        reduce(gy);
#pragma unroll
        for (int ib = 0; ib < NB; ++ib)
#pragma unroll
            for (int kb = 0; kb < NB; ++kb)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int r = 8 * ib + g, z = 8 * kb + c0 + e;
                    if (cw == 0 && r < R && z < R) yv[(int64_t)k * R * R + r * R + z] = gy[ib * NB + kb][e];
                }
        __syncwarp();
    }
}

// slices with more than max(512, 2 x mean) rows take the cooperative (CTA per slice) variant: it repeats the
// R x R serial part in every warp, so it only pays for the outliers that would otherwise set the kernel's tail
constexpr int kAlsLongRows = 512;

template <int NB>
int launch_als_polar_mma(dash_ctx *ctx, cudaStream_t st, const int64_t *row_ptr, const int64_t *row_ptr_host, int K,
                         const double *XV, const double *W, const double *H, int R, double *T, double *Q,
                         double *yv) {
    constexpr int NW = NB == 1 ? 8 : (NB == 2 ? 5 : 4);  // NB = 2: ~72 KB per CTA -> 3 CTAs = 15 warps per SM
    // long slices first (longest first), then the short ones in tensor order
    std::vector<int32_t> ord;
    ord.reserve(K);
    static const char *long_env = getenv("DASH_ALS_LONG");  // A/B: rows above which a slice takes the cooperative variant
    const int64_t long_rows = long_env ? atoll(long_env)
                                       : std::max<int64_t>(kAlsLongRows, 2 * (row_ptr_host[K] - row_ptr_host[0]) / std::max(K, 1));
    for (int k = 0; k < K; ++k)
        if (row_ptr_host[k + 1] - row_ptr_host[k] > long_rows) ord.push_back(k);
    const int nlong = (int)ord.size();
    std::stable_sort(ord.begin(), ord.end(), [row_ptr_host](int a, int b) {
        return row_ptr_host[a + 1] - row_ptr_host[a] > row_ptr_host[b + 1] - row_ptr_host[b];
    });
    for (int k = 0; k < K; ++k)
        if (row_ptr_host[k + 1] - row_ptr_host[k] <= long_rows) ord.push_back(k);
    if (ensure(ctx->items, sizeof(int32_t) * (size_t)std::max(K, 1))) return DASH_E_CUDA;
    int32_t *list = (int32_t *)ctx->items.p;
    // pageable source: the call returns once `ord` has been read into the driver's staging buffer
    cudaMemcpyAsync(list, ord.data(), sizeof(int32_t) * (size_t)K, cudaMemcpyHostToDevice, st);
    auto per_sm = [&](size_t smem) { return std::max<int>(1, (int)std::min<size_t>(8, (size_t)(227 * 1024) / (smem + 1024))); };
    // the long-slice kernel runs beside the short-slice one (disjoint slices and rows): both end in a
    // low-occupancy tail that the other can fill
    bool forked = false;
    if (nlong > 0) {
        const size_t smem = AlsMmaSmem<NB>::bytes(NW, true);
        ensure_smem_attr(k_als_polar_mma<NB, NW, true>, smem);
        cudaStream_t ls = st;
        if (K > nlong) {
            if (!ctx->aux_stream && (cudaStreamCreateWithFlags(&ctx->aux_stream, cudaStreamNonBlocking) != cudaSuccess ||
                                     cudaEventCreateWithFlags(&ctx->aux_fork, cudaEventDisableTiming) != cudaSuccess ||
                                     cudaEventCreateWithFlags(&ctx->aux_join, cudaEventDisableTiming) != cudaSuccess))
                return DASH_E_CUDA;
            cudaEventRecord(ctx->aux_fork, st);
            cudaStreamWaitEvent(ctx->aux_stream, ctx->aux_fork, 0);
            ls = ctx->aux_stream;
            forked = true;
        }
        k_als_polar_mma<NB, NW, true><<<std::min(nlong, ctx->num_sms * per_sm(smem)), NW * 32, smem, ls>>>(
            row_ptr, list, nlong, XV, W, H, R, T, Q, yv, ctx->err);
        if (forked) cudaEventRecord(ctx->aux_join, ls);
    }
    if (K > nlong) {
        const size_t smem = AlsMmaSmem<NB>::bytes(NW, false);
        ensure_smem_attr(k_als_polar_mma<NB, NW, false>, smem);
        const int ns = K - nlong;
        k_als_polar_mma<NB, NW, false><<<std::max(1, std::min((ns + NW - 1) / NW, ctx->num_sms * per_sm(smem))),
                                          NW * 32, smem, st>>>(row_ptr, list + nlong, ns, XV, W, H, R, T, Q, yv,
                                                               ctx->err);
    }
    if (forked) cudaStreamWaitEvent(st, ctx->aux_join, 0);
    return cudaGetLastError() == cudaSuccess ? 0 : DASH_E_CUDA;
}

// CP sweep on the projected tensor (als.py:166-176), a cooperative grid:
//   vtv = V^T V, wtw = W^T W, rhs_h = sum_k yv_k diag(W_k), H = ridge(vtv o wtw, rhs_h^T)^T,
//   hth = H^T H, rhs_w[k] = sum_r yv[k][r][:] o H[r][:], W = ridge(hth o vtv, rhs_w^T)^T,
//   wtw = W^T W.  Outputs H, W and lhs_v = hth o wtw (for the V solve).
// Each CTA owns a contiguous range of slices: it forms that range's partial sums, the grid
// syncs, and every CTA adds the partials in CTA order (identical bytes everywhere) and solves
// the two R x R systems redundantly; the per-slice W solves and the second partial wtw are
// again per range.  (One CTA looping over all K slices took 1.3 ms at the daily shape.)
template <int RB>
__global__ void __launch_bounds__(256) k_als_cp(const double *__restrict__ yv, int K, const double *__restrict__ V,
                                                int J, int R, double eps, double *__restrict__ H,
                                                double *__restrict__ W, double *__restrict__ lhs_v,
                                                double *__restrict__ part, unsigned long long *err) {
    constexpr int LD = RB + 1;
    cooperative_groups::grid_group grid = cooperative_groups::this_grid();
    const int G = gridDim.x, RR = R * R;
    const int kper = (K + G - 1) / G;
    const int k0 = min(K, (int)blockIdx.x * kper), k1 = min(K, k0 + kper);
    double *part1 = part;                        // [G][2][RR]: wtw, rhs_h partials
    double *part2 = part + (size_t)G * 2 * RR;   // [G][RR]: new wtw partials
    __shared__ double vtv[RB * LD], wtw[RB * LD], rh[RB * LD], Hn[RB * LD];
    double *hth = rh;  // rhs_h is dead once H is solved
    __shared__ double Ls[RB * LD], dinv[RB];
    __shared__ int piv[RB];
    __shared__ int okflag;
    const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
    for (int p = tid; p < R * R; p += blockDim.x) {
        const int r = p / R, z = p % R;
        double a = 0.0, b = 0.0, c = 0.0;
        for (int j = 0; j < J; ++j) a = fma(V[j * R + r], V[j * R + z], a);
        for (int k = k0; k < k1; ++k) b = fma(W[(int64_t)k * R + r], W[(int64_t)k * R + z], b);
        for (int k = k0; k < k1; ++k) c = fma(yv[(int64_t)k * R * R + r * R + z], W[(int64_t)k * R + z], c);
        vtv[r * LD + z] = a;
        part1[((size_t)blockIdx.x * 2 + 0) * RR + p] = b;
        part1[((size_t)blockIdx.x * 2 + 1) * RR + p] = c;
    }
    grid.sync();
    for (int p = tid; p < R * R; p += blockDim.x) {
        const int r = p / R, z = p % R;
        double b = 0.0, c = 0.0;
        for (int g = 0; g < G; ++g) {
            b += part1[((size_t)g * 2 + 0) * RR + p];
            c += part1[((size_t)g * 2 + 1) * RR + p];
        }
        wtw[r * LD + z] = b;
        rh[r * LD + z] = c;  // rhs_h[r][z]
    }
    __syncthreads();
    // generic: factor lhs (in Ls via warp 0), then solve `nrhs` systems; rhs column c, entry r
    auto factor = [&](auto lhs_of) {
        if (w == 0) {
            double tr = 0.0;
            for (int r = 0; r < R; ++r) tr += lhs_of(r, r);
            const double sh = eps * (tr / R);
            double row[RB];
#pragma unroll
            for (int z = 0; z < RB; ++z)
                row[z] = (lane < R && z < R) ? lhs_of(lane, z) + (lane == z ? sh : 0.0) : (lane == z ? 1.0 : 0.0);
            bool ok = chol_regs<RB>(row, Ls, LD, dinv);
            if (!ok && lane == 0) {
                for (int r = 0; r < R; ++r)
                    for (int z = 0; z < R; ++z) Ls[r * LD + z] = lhs_of(r, z) + (r == z ? sh : 0.0);
                if (!lu_factor_serial(Ls, LD, R, piv) && blockIdx.x == 0) report_error(err, -1, DASH_E_SINGULAR);
            }
            if (lane == 0) okflag = ok ? 1 : 0;
        }
        __syncthreads();
    };
    auto solve_one = [&](double (&b)[RB]) {
        if (okflag) {
            chol_solve_lane<RB>(Ls, LD, dinv, b);
        } else {
            double x[RB];  // rare LU path: local memory is fine
#pragma unroll
            for (int r = 0; r < RB; ++r) x[r] = b[r];
            lu_solve_serial(Ls, LD, R, piv, x);
#pragma unroll
            for (int r = 0; r < RB; ++r) b[r] = r < R ? x[r] : 0.0;
        }
    };
    // H = ridge(vtv o wtw, rhs_h^T)^T : system matrix symmetric; column c of rhs_h^T is row c of rhs_h
    factor([&](int r, int z) { return vtv[r * LD + z] * wtw[r * LD + z]; });
    if (tid < R) {
        double b[RB];
#pragma unroll
        for (int r = 0; r < RB; ++r) b[r] = r < R ? rh[tid * LD + r] : 0.0;  // rhs_h^T[:, c=tid] = rhs_h[tid][:]
        solve_one(b);
#pragma unroll
        for (int r = 0; r < RB; ++r)
            if (r < R) Hn[tid * LD + r] = b[r];  // H[tid][r] = x^T
    }
    __syncthreads();
    for (int p = tid; p < R * R; p += blockDim.x) {
        const int r = p / R, z = p % R;
        if (blockIdx.x == 0) H[p] = Hn[r * LD + z];
        double a = 0.0;
        for (int m = 0; m < R; ++m) a = fma(Hn[m * LD + r], Hn[m * LD + z], a);
        hth[r * LD + z] = a;
    }
    __syncthreads();
    // W = ridge(hth o vtv, rhs_w^T)^T, rhs_w[k][z] = sum_r yv[k][r][z] H[r][z]
    factor([&](int r, int z) { return hth[r * LD + z] * vtv[r * LD + z]; });
    for (int k = k0 + tid; k < k1; k += blockDim.x) {
        double b[RB];
#pragma unroll
        for (int z = 0; z < RB; ++z) {
            double a = 0.0;
            if (z < R)
                for (int r = 0; r < R; ++r) a = fma(yv[(int64_t)k * R * R + r * R + z], Hn[r * LD + z], a);
            b[z] = a;
        }
        solve_one(b);
        bool fin = true;
#pragma unroll
        for (int z = 0; z < RB; ++z)
            if (z < R) {
                W[(int64_t)k * R + z] = b[z];
                fin = fin && finite_d(b[z]);
            }
        if (!fin) report_error(err, k, DASH_E_NONFINITE);
    }
    __syncthreads();
    for (int p = tid; p < R * R; p += blockDim.x) {
        const int r = p / R, z = p % R;
        double b = 0.0;
        for (int k = k0; k < k1; ++k) b = fma(W[(int64_t)k * R + r], W[(int64_t)k * R + z], b);
        part2[(size_t)blockIdx.x * RR + p] = b;
    }
    grid.sync();
    if (blockIdx.x == 0)
        for (int p = tid; p < R * R; p += blockDim.x) {
            const int r = p / R, z = p % R;
            double b = 0.0;
            for (int g = 0; g < G; ++g) b += part2[(size_t)g * RR + p];
            lhs_v[p] = hth[r * LD + z] * b;
        }
}

// Z[row] = (Q[row] H) o w_k  (and, with w == nullptr, U = Q H)
__global__ void k_als_qh(const double *__restrict__ Q, const double *__restrict__ H, const double *__restrict__ W,
                         const int32_t *__restrict__ row_slice, int64_t N, int R, double *__restrict__ Z) {
    __shared__ double Hs[DASH_MAX_RANK * DASH_MAX_RANK];
    for (int i = threadIdx.x; i < R * R; i += blockDim.x) Hs[i] = H[i];
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N * R; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i / R;
        const int z = (int)(i % R);
        double a = 0.0;
        for (int r = 0; r < R; ++r) a = fma(Q[row * R + r], Hs[r * R + z], a);
        Z[i] = W ? a * W[(int64_t)row_slice[row] * R + z] : a;
    }
}

// per-slice sum of squared residuals ||X_k - Z_k V^T||^2 (warp per slice)
__global__ void __launch_bounds__(256) k_als_loss(const double *__restrict__ X, int64_t ldx,
                                                  const int64_t *__restrict__ row_ptr, int K,
                                                  const double *__restrict__ Z, const double *__restrict__ V, int J,
                                                  int R, double *__restrict__ per_slice) {
    const int lane = lane_id();
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    __shared__ double zs_s[8][DASH_MAX_RANK];
    double *zs = zs_s[warp_id()];
    for (int k = gw; k < K; k += nw) {
        const int64_t r0 = row_ptr[k], r1 = row_ptr[k + 1];
        double acc = 0.0;
        for (int64_t row = r0; row < r1; ++row) {
            if (lane < R) zs[lane] = Z[row * R + lane];
            __syncwarp();
            for (int j = lane; j < J; j += 32) {
                double rec = 0.0;
                for (int r = 0; r < R; ++r) rec = fma(zs[r], __ldg(V + (int64_t)j * R + r), rec);
                const double d = X[row * ldx + j] - rec;
                acc = fma(d, d, acc);
            }
            __syncwarp();
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(FULL_MASK, acc, off);
        if (lane == 0) per_slice[k] = acc;
    }
}

__global__ void k_sum_ordered(const double *__restrict__ v, int n, double *__restrict__ out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double acc = 0.0;
        for (int i = 0; i < n; ++i) acc += v[i];
        *out = acc;
    }
}

template <int RB>
int launch_als_polar(dash_ctx *ctx, cudaStream_t st, const int64_t *row_ptr, int K, const double *XV,
                     const double *W, const double *H, int R, double *T, double *Q, double *yv) {
    constexpr int NW = RB <= 16 ? 4 : 2;
    const size_t smem = AlsSmem<RB>::bytes(NW);
    ensure_smem_attr(k_als_polar<RB, NW>, smem);
    const int blocks = std::max(1, std::min((K + NW - 1) / NW, ctx->num_sms * 8));
    k_als_polar<RB, NW><<<blocks, NW * 32, smem, st>>>(row_ptr, K, XV, W, H, R, T, Q, yv, ctx->err);
    return 0;
}

template <int RB>
int launch_als_cp(dash_ctx *ctx, cudaStream_t st, const double *yv, int K, const double *V, int J, int R, double eps,
                  double *H, double *W, double *lhs_v, unsigned long long *err) {
    // ranges of >= 32 slices, at most one CTA per SM (cooperative launch: all CTAs co-resident)
    const int G = std::max(1, std::min(ctx->num_sms, (K + 31) / 32));
    if (ensure(ctx->part, sizeof(double) * (size_t)G * 3 * R * R)) return DASH_E_CUDA;
    double *part = (double *)ctx->part.p;
    void *args[] = {(void *)&yv, (void *)&K, (void *)&V, (void *)&J, (void *)&R, (void *)&eps, (void *)&H,
                    (void *)&W, (void *)&lhs_v, (void *)&part, (void *)&err};
    return cudaLaunchCooperativeKernel((const void *)k_als_cp<RB>, dim3(G), dim3(256), args, 0, st) == cudaSuccess
               ? 0 : DASH_E_CUDA;
}

}  // namespace

extern "C" {

int dash_als_sweep_f64(dash_ctx *ctx, void *stream, const dash_batch_f64 *t, int32_t J, int32_t R, double *V,
                       double *H, double *W, double *Q, double *loss, double eps) {
    if (!ctx || !t || R < 1 || R > DASH_MAX_RANK_ALS || J < 1 || t->M < 1) return DASH_E_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    ctx->last_launches = 0;
    const int K = t->M;
    const int64_t N = t->N;
    const int RB = rank_bucket(R);
    int64_t nsplit, rps;
    plan_fsplit(ctx, N, J, nsplit, rps);
    if (ensure(ctx->xv, sizeof(double) * N * R) || ensure(ctx->row_slice, sizeof(int32_t) * N) ||
        ensure(ctx->fslots, sizeof(double) * nsplit * J * R) || ensure(ctx->fg, sizeof(double) * ((size_t)J * R + R * R)) ||
        ensure(ctx->scratch, sizeof(double) * ((size_t)N * R * 2 + (size_t)K * R * R + K + R * R + 8) +
                                 sizeof(int32_t) * K))
        return DASH_E_CUDA;
    double *XV = (double *)ctx->xv.p;
    int32_t *row_slice = (int32_t *)ctx->row_slice.p;
    double *T = (double *)ctx->scratch.p;
    double *Z = T + (size_t)N * R;
    double *yv = Z + (size_t)N * R;
    double *per = yv + (size_t)K * R * R;
    double *lhs_v = per + K;
    int32_t *ident = (int32_t *)(lhs_v + R * R + 8);
    std::vector<int32_t> id(K);
    for (int i = 0; i < K; ++i) id[i] = i;
    cudaMemcpyAsync(ident, id.data(), sizeof(int32_t) * K, cudaMemcpyHostToDevice, st);
    dash_batch_f64 b = *t;
    b.state_row = ident;
    k_row_slice<<<std::min(ctx->num_sms * 4, (K + 7) / 8 + 1), 256, 0, st>>>(t->row_ptr, K, row_slice);
    // the two streaming contractions take the update path's tensor-map kernels when the shape allows
    // (R bucket 16 and even, J <= 128: k_xv3 / k_fgemm3; J > 128: k_xvw / k_fgemmw), else the generic ones
    const bool tma = N > 0 && tma_ok(&b, J, R) && !ensure(ctx->vtv, sizeof(double) * R * R) &&
                     !ensure(ctx->fsnap, sizeof(double) * J * R) && !ensure(ctx->gsnap, sizeof(double) * R * R);
    const bool wide = !tma && N > 0 && widej_ok(&b, J, R, V);
    if (tma) {
        nsplit = ctx->num_sms;  // one F slot per CTA
    } else if (wide) {
        const int fc = RB <= 32 ? WideCfg<32>::FC : WideCfg<64>::FC;
        ctx->wnj = (J + fc - 1) / fc;
        const int64_t nrow = std::max<int64_t>(1, ctx->num_sms / ctx->wnj);
        ctx->rps = std::max<int64_t>(32, ((N + nrow - 1) / nrow + 31) / 32 * 32);
        ctx->nsplit = nsplit = (N + ctx->rps - 1) / ctx->rps;
    }
    if ((tma || wide) && ensure(ctx->fslots, sizeof(double) * nsplit * J * R)) return DASH_E_CUDA;
    if (tma) {
        const FusedPrologue pro{(double *)ctx->vtv.p, V, V, (double *)ctx->fsnap.p, (double *)ctx->gsnap.p,
                                (double *)ctx->fsnap.p, 0, 0};  // only vtv is produced (unused here)
        if (launch_xv3(ctx, st, &b, J, V, R, XV, pro, false)) return DASH_E_CUDA;
    } else if (wide) {
        if (launch_xvw(ctx, st, &b, J, V, R, XV)) return DASH_E_CUDA;
    } else {
        launch_xv(ctx, st, &b, J, V, R, XV);
    }
    static const bool polar_scalar = getenv("DASH_ALS_POLAR_SCALAR") != nullptr;  // A/B switch
    if (!polar_scalar) {
        int rc_p;
        switch (RB) {
            case 4:
            case 8: rc_p = launch_als_polar_mma<1>(ctx, st, t->row_ptr, t->row_ptr_host, K, XV, W, H, R, T, Q, yv); break;
            case 16: rc_p = launch_als_polar_mma<2>(ctx, st, t->row_ptr, t->row_ptr_host, K, XV, W, H, R, T, Q, yv); break;
            default: rc_p = launch_als_polar_mma<4>(ctx, st, t->row_ptr, t->row_ptr_host, K, XV, W, H, R, T, Q, yv); break;
        }
        if (rc_p) return rc_p;
    } else
    switch (RB) {
        case 4: launch_als_polar<4>(ctx, st, t->row_ptr, K, XV, W, H, R, T, Q, yv); break;
        case 8: launch_als_polar<8>(ctx, st, t->row_ptr, K, XV, W, H, R, T, Q, yv); break;
        case 16: launch_als_polar<16>(ctx, st, t->row_ptr, K, XV, W, H, R, T, Q, yv); break;
        default: launch_als_polar<32>(ctx, st, t->row_ptr, K, XV, W, H, R, T, Q, yv); break;
    }
    int rc_cp;
    switch (RB) {
        case 4: rc_cp = launch_als_cp<4>(ctx, st, yv, K, V, J, R, eps, H, W, lhs_v, ctx->err); break;
        case 8: rc_cp = launch_als_cp<8>(ctx, st, yv, K, V, J, R, eps, H, W, lhs_v, ctx->err); break;
        case 16: rc_cp = launch_als_cp<16>(ctx, st, yv, K, V, J, R, eps, H, W, lhs_v, ctx->err); break;
        default: rc_cp = launch_als_cp<32>(ctx, st, yv, K, V, J, R, eps, H, W, lhs_v, ctx->err); break;
    }
    if (rc_cp) return rc_cp;
    const int qb = (int)std::min<int64_t>((N * R + 255) / 256, (int64_t)ctx->num_sms * 16);
    // rhs_v = X^T ((Q H) o w).  Tensor-map paths: Z = (Q H) o w once (the loss below reads the same Z);
    // generic path: the F GEMM multiplies "U" = Q H by W[state_row[slice]] itself
    k_als_qh<<<std::max(qb, 1), 256, 0, st>>>(Q, H, (tma || wide) ? W : nullptr, row_slice, N, R, Z);
    if (tma) {
        if (launch_f3(ctx, st, &b, J, Z, R, (double *)ctx->fslots.p)) return DASH_E_CUDA;
    } else if (wide) {
        if (launch_fw(ctx, st, &b, J, Z, R, (double *)ctx->fslots.p, nullptr)) return DASH_E_CUDA;
    } else {
        launch_fgemm(ctx, st, &b, J, Z, row_slice, W, R, rps, (int)nsplit, (double *)ctx->fslots.p);
    }
    if (colsum(ctx, st, (double *)ctx->fslots.p, (int)nsplit, (int64_t)J * R, (double *)ctx->fg.p))
        return DASH_E_CUDA;
    // V = ridge(lhs_v, rhs_v^T)^T  (rhs_v^T (R x J): entry (r, j) = rhs_v[j][r])
    switch (RB) {
        case 4: k_ridge<4><<<1, 32, 0, st>>>(lhs_v, (double *)ctx->fg.p, R, J, 1, R, eps, V, ctx->err); break;
        case 8: k_ridge<8><<<1, 32, 0, st>>>(lhs_v, (double *)ctx->fg.p, R, J, 1, R, eps, V, ctx->err); break;
        case 16: k_ridge<16><<<1, 32, 0, st>>>(lhs_v, (double *)ctx->fg.p, R, J, 1, R, eps, V, ctx->err); break;
        default: k_ridge<32><<<1, 32, 0, st>>>(lhs_v, (double *)ctx->fg.p, R, J, 1, R, eps, V, ctx->err); break;
    }
    // loss with the refreshed H, W, V (als.py:182-185): Z = (Q H) o w
    if (!(tma || wide)) k_als_qh<<<std::max(qb, 1), 256, 0, st>>>(Q, H, W, row_slice, N, R, Z);
    if (ensure(ctx->rerr, sizeof(double) * (size_t)N)) return DASH_E_CUDA;
    launch_row_err<false>(ctx, st, t->X, t->ldx, N, (const double *)Z, R, V, J, (const int32_t *)nullptr,
                          (const int32_t *)nullptr, (const double *)nullptr, (double *)ctx->rerr.p);
    k_seg_sum<<<std::max(1, std::min((K + 7) / 8, ctx->num_sms * 8)), 256, 0, st>>>((const double *)ctx->rerr.p,
                                                                                  t->row_ptr, K, J, 0, per);
    k_tree_sum<<<1, kTreeThreads, 0, st>>>(per, K, 0, loss);
    return cudaGetLastError() == cudaSuccess ? DASH_OK : DASH_E_CUDA;
}

int dash_als_project_f64(dash_ctx *ctx, void *stream, int64_t N, int32_t R, const double *Q, const double *H,
                         double *U) {
    if (!ctx || R < 1 || R > DASH_MAX_RANK || N < 0) return DASH_E_ARG;
    if (N == 0) return DASH_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int qb = (int)std::min<int64_t>((N * R + 255) / 256, (int64_t)ctx->num_sms * 16);
    k_als_qh<<<std::max(qb, 1), 256, 0, st>>>(Q, H, nullptr, nullptr, N, R, U);
    return cudaGetLastError() == cudaSuccess ? DASH_OK : DASH_E_CUDA;
}

}  // extern "C"
