// k_big: the per-slice phase for BIG slices (> kSmallRows rows), R <= 16,
// one CTA (8 warps) per slice, the row work on the FP64 tensor pipe:
//
//   M      = -A^{-1} diag(s)          (group sweep, warp 0)        _kernels.py:86-97
//   per 64-row block of XV (cp.async double-buffered):
//     U    = XV M^T        (DMMA 64x16x16)  -> U_out               _kernels.py:97-101
//     c   += diag(XV^T U)  (fragment FMAs)                         _kernels.py:104-108
//     gram+= U^T U         (DMMA 16x16x64)                          _kernels.py:109-115
//   w = B^{-1} c_new, B = vtv o (lam D + gram) + shift (group sweep, warp 0)
//   US = U o w  (L2-hot re-read of the rows just written), G slot = gram o w w^T.
//
// The reference sums c / gram row by row; here the sums run in DMMA / block
// order (fixed -> deterministic; differences are rounding-level).
// (included inside dash_update.cu's anonymous namespace)
#pragma once

struct BigSmem {
    static constexpr int RB = 16, RP = 16;
    static constexpr int BR = 64;           // rows per block
    static constexpr int XPI = RP + 4;      // XV staging pitch (A-frag reads conflict-free)
    static constexpr int UPI = RP + 8;      // U block pitch (gram frags conflict-free)
    static constexpr int MPI = RP + 4;      // M pitch (B-frag reads)
    static constexpr int LDV = RB + 2;
    static constexpr int LDL = RB + 1;
    static constexpr int NS = 3;            // XV staging ring depth
    // xs[NS][BR*XPI] | us[BR*UPI] | Ms[RP*MPI] | vtv[RB*LDV] | red[8*64] | gram_s[RB*LDL] | buf[RB] | dn[RB*LDL]
    // | lu[RB*LDL] | vec[4*RB] | piv[RB]
    static constexpr int doubles =
        NS * BR * XPI + BR * UPI + RP * MPI + RB * LDV + 8 * 64 + RB * LDL + RB + RB * LDL + RB * LDL + 4 * RB + RB;
    static constexpr size_t bytes() { return sizeof(double) * doubles + 64; }
};

__device__ __forceinline__ void cp_async16(double *dst, const double *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }
__device__ __forceinline__ void cp_async_wait2() { asm volatile("cp.async.wait_group 2;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

// stage XV rows [row0, row0+nr) into xs (pitch XPI); R must be even (16-byte chunks)
__device__ __forceinline__ void big_stage(double *xs, const double *XV, int64_t row0, int nr, int R) {
    using B = BigSmem;
    const int chunks = R / 2;
    for (int e = threadIdx.x; e < B::BR * chunks; e += blockDim.x) {
        const int i = e / chunks, c2 = e % chunks;
        if (i < nr) cp_async16(xs + i * B::XPI + 2 * c2, XV + (row0 + i) * R + 2 * c2);
    }
}

// CTA b processes big slices b, b + gridDim.x, ... of the device plan (meta +
// nsmall, longest size class first; launched with one CTA per big slice) and
// accumulates their gram o w w^T into its own G slot (deterministic).
__global__ void __launch_bounds__(256, 2) k_big(SliceParams p, const int4 *__restrict__ meta,
                                                const int *__restrict__ plan_counts) {
    using B = BigSmem;
    constexpr int RB = B::RB, RP = B::RP, BR = B::BR, XPI = B::XPI, UPI = B::UPI, MPI = B::MPI, LDV = B::LDV,
                  LDL = B::LDL;
    extern __shared__ __align__(16) double sm[];
    double *xs0 = sm;
    double *us = xs0 + B::NS * BR * XPI;
    double *Ms = us + BR * UPI;
    double *vtv_s = Ms + RP * MPI;
    double *red = vtv_s + RB * LDV;      // 8 warps x 64
    double *gram_s = red + 8 * 64;
    double *buf = gram_s + RB * LDL;
    double *dns = buf + RB;
    double *lu = dns + RB * LDL;
    double *vec = lu + RB * LDL;         // s | c | w | spare
    int *piv = reinterpret_cast<int *>(vec + 4 * RB);
    const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
    const int g = lane >> 2, t = lane & 3;
    const int R = p.R;
    // PDL: launched behind the small-slice kernel, whose CTAs trigger only
    // after their own pdl_wait -- so XV, vtv and the plan are complete here.
    // The two kernels touch disjoint slices / rows / G slots, so this one does
    // not wait for the small-slice kernel until it exits (tail overlap).
    // Its own dependent (the F GEMM) is released only once every CTA is past
    // its row pass: a successor made resident earlier would hold shared
    // memory the remaining big / small slices need (measured: the FP32 data
    // mode's 83 KB F-GEMM CTAs, which fit beside k_big, cost 160 us/update).
    const int nsmall = __ldcg(plan_counts), nbig = __ldcg(plan_counts + 1);
    for (int i = tid; i < RB * LDV; i += blockDim.x) {
        const int a = i / LDV, b = i % LDV;
        vtv_s[i] = (a < R && b < R) ? __ldcg(p.vtv + a * R + b) : 0.0;  // L2: written by the XV kernel
    }
    double gslot = 0.0;  // this thread's entry (tid) of the CTA's G slot
    for (int bi = blockIdx.x; bi < nbig; bi += gridDim.x) {
        __syncthreads();  // previous slice done with the shared buffers
        const int4 mt = __ldcg(meta + nsmall + bi);
        const int m = mt.w;
        const int64_t r0 = mt.x, n = mt.y;
        const int wrow = mt.z & 0x7fffffff;
        const bool fresh = mt.z < 0;
        // prefetch the first two XV blocks while the A system is solved
        const int nblk = (int)((n + BR - 1) / BR);
        for (int q = 0; q < B::NS - 1; ++q) {
            if (q < nblk) big_stage(xs0 + q * BR * XPI, p.XV, r0 + (int64_t)q * BR, (int)min((int64_t)BR, n - (int64_t)q * BR), R);
            cp_async_commit();
        }
        if (tid < RB) vec[tid] = tid < R ? ((fresh && p.pass == 0) ? 1.0 : __ldcg(p.W + (int64_t)wrow * R + tid)) : 0.0;
        if (tid < RB && !fresh)
            for (int z = 0; z < R; ++z) dns[tid * LDL + z] = tid < R ? __ldcg(p.D + (int64_t)wrow * R * R + (int64_t)z * R + tid) : 0.0;
        const double cold = (tid < R && !fresh) ? __ldcg(p.C + (int64_t)wrow * R + tid) : 0.0;
        __syncthreads();
        // ---- A sweep by warp 0, lanes 0..15 (lanes 16..31 run a harmless identity copy)
        if (w == 0) {
            // s is read from shared (vec) rather than held in a register array: keeps
            // the sweep's live set at a[] + the gathered column (no spills)
            const int r = lane % RB;
            const bool real = lane < RB && r < R;
            const double s_r = real ? vec[r] : 0.0;
            double sh = 0.0;
    #pragma unroll
            for (int z = 0; z < RB; ++z)
                if (z < R) sh += vtv_s[z * LDV + z] * vec[z] * vec[z];
            sh = p.eps * sh / R;
            const double dg = real ? sh : 1.0;
            const double *vrow = vtv_s + r * LDV;
            double a2[RB];
    #pragma unroll
            for (int z = 0; z < RB; ++z) a2[z] = (lane < RB ? vrow[z] * s_r * vec[z] : 0.0) + ((z == r) ? dg : 0.0);
            // lanes 0..15 sweep A; lanes 16..31 sweep a harmless identity (own gather buffer)
            const bool okA = sweep_inverse<RB>(a2, lane < RB ? buf : red + 7 * 64, r);
            const unsigned badA = __ballot_sync(FULL_MASK, !okA) & 0xffffu;
            if (badA) {
                const bool need = lane < RB;
    #pragma unroll
                for (int z = 0; z < RB; ++z)
                    if (need) a2[z] = vrow[z] * s_r * vec[z] + ((z == r) ? dg : 0.0);
                if (lane == 0) atomicAdd(p.fallbacks, 1u);
                const bool okLU = lu_fallback<RB>(a2, lu, piv, r, R, need);
                if (lane == 0 && !okLU) report_error(p.err, m, DASH_E_SINGULAR);
            }
            // Ms[n][k] = A^{-1}[n][k] s_k, so U = XV Ms^T  (a2 holds -A^{-1})
            if (lane < RB) {
    #pragma unroll
                for (int z = 0; z < RB; ++z) Ms[r * MPI + z] = -a2[z] * vec[z];
            }
        }
        __syncthreads();

        // ---- rows, one 64-row block at a time (double-buffered XV)
        double cacc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};  // c partials for cols (nb*8 + 2t + e)
        double gacc[2] = {0.0, 0.0};  // gram tile (mi, ni) = ((w&3) >> 1, w & 1), K half w >> 2
        for (int bi = 0; bi < nblk; ++bi) {
            double *xs = xs0 + (bi % B::NS) * BR * XPI;
            const int64_t b0 = r0 + (int64_t)bi * BR;
            const int nr = (int)min((int64_t)BR, n - (int64_t)bi * BR);
            {
                const int q = bi + B::NS - 1;  // refill the stage consumed two blocks ago
                if (q < nblk)
                    big_stage(xs0 + (q % B::NS) * BR * XPI, p.XV, r0 + (int64_t)q * BR,
                              (int)min((int64_t)BR, n - (int64_t)q * BR), R);
                cp_async_commit();
            }
            cp_async_wait2();
            __syncthreads();
            if (nr < BR || R < RP) {  // zero padded columns / tail rows of the staged block
                for (int e = tid; e < BR * XPI; e += blockDim.x) {
                    const int i = e / XPI, z = e % XPI;
                    if (i >= nr || z >= R) xs[e] = 0.0;
                }
                __syncthreads();
            }
            // U = XV Ms^T: warp w -> rows 8w..8w+7, both n-tiles
            double uacc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    #pragma unroll
            for (int kk = 0; kk < RP / 4; ++kk) {
                const double a = xs[(8 * w + g) * XPI + 4 * kk + t];
    #pragma unroll
                for (int nb = 0; nb < 2; ++nb) dmma884(uacc[nb], a, Ms[(8 * nb + g) * MPI + 4 * kk + t]);
            }
            const int row = 8 * w + g;
    #pragma unroll
            for (int nb = 0; nb < 2; ++nb)
    #pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int col = 8 * nb + 2 * t + e;
                    const double u = (row < nr && col < R) ? uacc[nb][e] : 0.0;
                    us[row * UPI + col] = u;
                    if (row < nr && col < R) p.U[(b0 + row) * R + col] = u;
                    cacc[nb][e] = fma(xs[row * XPI + col], u, cacc[nb][e]);
                }
            __syncthreads();
            // gram += U^T U : 8 warps = 4 tiles x 2 K-halves (8-deep DMMA chains)
            {
                const int mi = (w & 3) >> 1, ni = w & 1, kh = w >> 2;
    #pragma unroll
                for (int kk = 0; kk < BR / 8; ++kk) {
                    const int row = 4 * (kk + kh * (BR / 8)) + t;
                    const double a = us[row * UPI + 8 * mi + g];
                    const double b = us[row * UPI + 8 * ni + g];
                    dmma884(gacc, a, b);
                }
            }
            __syncthreads();
        }
        // ---- reduce c (over lanes g and warps) and gram tiles into shared
    #pragma unroll
        for (int nb = 0; nb < 2; ++nb)
    #pragma unroll
            for (int e = 0; e < 2; ++e) {
                double v = cacc[nb][e];
                v += __shfl_xor_sync(FULL_MASK, v, 4);
                v += __shfl_xor_sync(FULL_MASK, v, 8);
                v += __shfl_xor_sync(FULL_MASK, v, 16);
                cacc[nb][e] = v;
            }
        if (g == 0) {
    #pragma unroll
            for (int nb = 0; nb < 2; ++nb)
    #pragma unroll
                for (int e = 0; e < 2; ++e) red[w * 64 + 8 * nb + 2 * t + e] = cacc[nb][e];
        }
        {
            const int mi = (w & 3) >> 1, ni = w & 1;
            if (w >= 4) {
    #pragma unroll
                for (int e = 0; e < 2; ++e) gram_s[(8 * mi + g) * LDL + 8 * ni + 2 * t + e] = gacc[e];
            }
            __syncthreads();
            if (w < 4) {  // fixed order: (first K half) + (second K half)
    #pragma unroll
                for (int e = 0; e < 2; ++e) {
                    double *gp = gram_s + (8 * mi + g) * LDL + 8 * ni + 2 * t + e;
                    *gp = gacc[e] + *gp;
                }
            }
        }
        __syncthreads();
        if (tid < RB) {
            double cs = 0.0;
            for (int ww = 0; ww < 8; ++ww) cs += red[ww * 64 + tid];
            vec[RB + tid] = tid < R ? p.lam * cold + cs : 0.0;  // c_new
        }
        pdl_trigger();
        __syncthreads();
        // ---- D accumulation and the S-row system by warp 0 lanes 0..15 (D row in shared dns)
        if (w == 0) {
            const int r = lane % RB;
            const bool lreal = lane < RB && r < R;
            double *dn = dns + r * LDL;
            if (lane < RB) {
    #pragma unroll
                for (int z = 0; z < RB; ++z)
                    dn[z] = (lreal && z < R) ? p.lam * (fresh ? 0.0 : dn[z]) + gram_s[r * LDL + z] : 0.0;
            }
            __syncwarp();
            double dsum = 0.0;
    #pragma unroll
            for (int z = 0; z < RB; ++z)
                if (z < R) dsum += vtv_s[z * LDV + z] * dns[z * LDL + z];
            const double sh2 = p.eps * dsum / R;
            const double dg2 = lreal ? sh2 : 1.0;
            double a[RB];
    #pragma unroll
            for (int z = 0; z < RB; ++z) a[z] = (lane < RB ? vtv_s[r * LDV + z] * dn[z] : 0.0) + ((z == r) ? dg2 : 0.0);
            double wv;  // w = B^{-1} c  (lu: scratch until a fallback; lanes 16..31 solve a harmless identity)
            bool okB = gj_solve<RB>(a, lreal ? vec[RB + r] : 0.0, lane < RB ? lu : red + 7 * 64, r, wv);
            if (!lreal) wv = 0.0;
            const bool good = __all_sync(FULL_MASK, (okB && isfinite(wv)) || lane >= RB);
            if (!good) {
                const bool need = lane < RB;
    #pragma unroll
                for (int z = 0; z < RB; ++z) a[z] = (lane < RB ? vtv_s[r * LDV + z] * dn[z] : 0.0) + ((z == r) ? dg2 : 0.0);
                if (lane == 0) atomicAdd(p.fallbacks, 1u);
                const bool okLU = lu_fallback<RB>(a, lu, piv, r, R, need);
                if (lane == 0 && !okLU) report_error(p.err, m, DASH_E_SINGULAR);
                wv = 0.0;
    #pragma unroll
                for (int z = 0; z < RB; ++z) wv = fma(-a[z], vec[RB + z], wv);
                if (!lreal) wv = 0.0;
                if (lreal && !isfinite(wv)) report_error(p.err, m, DASH_E_NONFINITE);
            }
            if (lreal) {
                p.W[(int64_t)wrow * R + r] = wv;
                if (p.final_pass) {
                    p.C[(int64_t)wrow * R + r] = vec[RB + r];
    #pragma unroll
                    for (int z = 0; z < RB; ++z)
                        if (z < R) p.D[(int64_t)wrow * R * R + (int64_t)z * R + r] = dn[z];
                }
            }
            if (lane < RB) vec[2 * RB + lane] = lreal ? wv : 0.0;
        }
        __syncthreads();
        // ---- G slot (gram o w w^T) and US = U o w (rows just written: L2-hot)
        if (tid < R * R) {
            const int a = tid / R, b = tid % R;
            gslot += gram_s[a * LDL + b] * vec[2 * RB + a] * vec[2 * RB + b];
        }
        if (p.US != nullptr) {
            // 16-byte chunks (R even); a thread's column pair advances by a fixed step
            // per iteration, so no per-element division.  Loads are batched ahead of
            // the stores (U and US never alias).
            const int half = R / 2;
            const int64_t tot = n * half;
            const double2 *__restrict__ Ur = reinterpret_cast<const double2 *>(p.U + r0 * R);
            double2 *__restrict__ USr = reinterpret_cast<double2 *>(p.US + r0 * R);
            const double *wv = vec + 2 * RB;
            const int step = blockDim.x % half;
            int col = tid % half;
            constexpr int UNR = 2;
            for (int64_t e0 = tid; e0 < tot; e0 += (int64_t)UNR * blockDim.x) {
                double2 v[UNR];
                int cc[UNR];
    #pragma unroll
                for (int k = 0; k < UNR; ++k) {
                    const int64_t e = e0 + (int64_t)k * blockDim.x;
                    if (e < tot) v[k] = __ldcg(Ur + e);
                    cc[k] = col;
                    col += step;
                    if (col >= half) col -= half;
                }
    #pragma unroll
                for (int k = 0; k < UNR; ++k) {
                    const int64_t e = e0 + (int64_t)k * blockDim.x;
                    if (e < tot) USr[e] = make_double2(v[k].x * wv[2 * cc[k]], v[k].y * wv[2 * cc[k] + 1]);
                }
            }
        }
        cp_async_wait_all();
    }  // big slices of this CTA
    if (tid < R * R) p.G_slots[(int64_t)blockIdx.x * R * R + tid] = gslot;
    pdl_wait();  // completion of this grid implies completion of the small-slice kernel
}

int launch_big(cudaStream_t st, int grid, const SliceParams &sp, const int4 *meta, const int *plan_counts) {
    const size_t smem = BigSmem::bytes();
    ensure_smem_attr(k_big, smem);
    return launch_k(pdl_site("big"), k_big, grid, 256, smem, st, sp, meta, plan_counts);
}
