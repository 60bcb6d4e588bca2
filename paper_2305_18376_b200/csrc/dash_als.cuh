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
    static constexpr int NRL = (NQ + 31) / 32;  // values per lane in the cross-warp reduction buffer
    // + red[nw][32 * NRL]: per-warp Gram partials, summed in warp order by every warp
    __host__ __device__ static constexpr size_t bytes(int nw) {
        return sizeof(double) * (shared + nw * per_warp + nw * 32 * NRL);
    }
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
    double *red = sm + S::shared + NW * S::per_warp;
    // Gram partials of the CTA's warps -> every warp holds the full sum (fixed warp order)
    auto reduce = [&](auto &acc) {
        constexpr int n = (int)(sizeof(acc) / sizeof(double));
#pragma unroll
        for (int q = 0; q < n; ++q) red[(w * S::NRL + q) * 32 + lane] = acc[q];
        __syncthreads();
#pragma unroll
        for (int q = 0; q < n; ++q) {
            double t = 0.0;
            for (int ww = 0; ww < NW; ++ww) t += red[(ww * S::NRL + q) * 32 + lane];
            acc[q] = t;
        }
        __syncthreads();
    };
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
    // one CTA per slice: its warps take the slice's 32-row chunks in turn (a single warp per slice
    // made the kernel as slow as its longest slice: 4,000 rows = 375 serial chunk passes)
    for (int k = blockIdx.x; k < K; k += gridDim.x) {
        const int64_t r0 = row_ptr[k], r1 = row_ptr[k + 1];
        if (lane < RB) wv[lane] = lane < R ? W[(int64_t)k * R + lane] : 0.0;
        __syncwarp();
        // ---- pass 1: T rows (als.py:156) and S1 = T^T T
        double g1[NPL];
#pragma unroll
        for (int q = 0; q < NPL; ++q) g1[q] = 0.0;
        for (int64_t c0 = r0 + 32 * w; c0 < r1; c0 += 32 * NW) {
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
        reduce(g1);
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
        for (int64_t c0 = r0 + 32 * w; c0 < r1; c0 += 32 * NW) {
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
        reduce(g2);
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
        if (!ok && lane == 0 && w == 0) report_error(err, k, DASH_E_SINGULAR);
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
        for (int64_t c0 = r0 + 32 * w; c0 < r1; c0 += 32 * NW) {
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
        reduce(gy);
#pragma unroll
        for (int q = 0; q < NQL; ++q) {
            const int pp = lane + 32 * q;
            if (pp < NQ && w == 0) {
                const int r = pa[NP + pp], z = pc[NP + pp];
                if (r < R && z < R) yv[(int64_t)k * R * R + r * R + z] = gy[q];
            }
        }
        __syncwarp();
    }
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
    const int blocks = std::max(1, std::min(K, ctx->num_sms * 8));
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
    k_tree_sum<<<1, 256, 0, st>>>(per, K, 0, loss);
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
