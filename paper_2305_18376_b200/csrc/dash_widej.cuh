// Wide-J streaming GEMMs (J > 128, any rank bucket up to 64; FP64 batches).
//
// The two contractions of stream.py:314-315 / :321 at BASELINE's "wide"
// shapes (J = 1,024, R in {10, 32, 64}).  A 32-row tile of X no longer fits a
// ring stage (256 KB), so both kernels chunk the long dimension and stream
// (X chunk, small-operand chunk) pairs through one TMA ring:
//
//   k_xvw<RP>    XV = X V.  Persistent CTAs take 64-row tiles; per 64-column
//                chunk a stage holds 8 X boxes (16 doubles x 32 rows, 128B
//                swizzle) and RP/16 boxes of V (16 ranks x 64 columns, same
//                swizzle) -- V is re-read from L2 once per 64 rows.  8 DMMA
//                warps as a 4 x 2 grid, each 16 rows x RP/2 ranks; A pairs by
//                LDS.128 (even / odd column of a pair = two k-steps), B by
//                LDS.64 from the swizzled [k][n] box (conflict-free: the four
//                k rows of a fragment are 2 apart, so their XOR patterns are
//                disjoint).
//   k_fgemmw<RP> F slot = X^T US over a row range, for a block of FC columns (256;
//                128 at RP = 64): grid = ceil(J / FC) column blocks x row ranges,
//                accumulators (FC x RP per CTA) stay in registers for the whole range, so
//                X is still read once; US (N x R) is re-read per column block
//                (L2).  Optional G slot = US^T US (k_slicesw's fresh G term),
//                its 8 x 8 tiles spread over the column blocks' warps.
//
// Rows past N and columns past J / R are zero-filled by TMA.
// (included inside dash_update.cu's anonymous namespace)
#pragma once

template <int RP>
struct WideCfg {
    static constexpr int NV = RP / 16;                   // 16-rank boxes of V / US
    static constexpr int XC = 64;                        // columns per XV chunk
    static constexpr int XV_SD = 8 * 512 + NV * 1024;    // stage doubles: X 64 x 64, V 64 x RP
    static constexpr int XV_ST = RP <= 16 ? 5 : (RP <= 32 ? 4 : 3);
    static constexpr int FC = RP <= 32 ? 256 : 128;      // columns per F column block (accumulators: FC x RP per CTA)
    static constexpr int FS = FC / 16;                   // strips per column block
    static constexpr int MAXS = FS / kCW;                // strips per warp
    static constexpr int F_SD = (FS + NV) * 512;         // stage doubles: X 32 x FC, US 32 x RP
    static constexpr int F_ST = RP <= 32 ? 3 : 4;
    static constexpr int GT = 2;                         // G tiles (8 x 8) per warp: needs (RP/8)^2 <= 16 nJ
    static constexpr size_t xv_bytes() { return 1024 + sizeof(double) * XV_ST * XV_SD + 16 * XV_ST; }
    static constexpr size_t f_bytes() { return 1024 + sizeof(double) * F_ST * F_SD + 16 * F_ST; }
};

template <int RP>
__global__ void __launch_bounds__(kCW * 32 + 32, 1) k_xvw(const __grid_constant__ CUtensorMap tmX,
                                                          const __grid_constant__ CUtensorMap tmV, int64_t N, int J,
                                                          int R, double *__restrict__ XV) {
    using C = WideCfg<RP>;
    constexpr int NBW = RP / 16;  // 8-rank blocks per warp
    extern __shared__ __align__(16) double sm_raw[];
    double *sm = align1k(sm_raw);
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + C::XV_ST * C::XV_SD);
    uint64_t *empty = full + C::XV_ST;
    const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
    const int g = lane >> 2, t = lane & 3;
    if (tid == 0) {
        prefetch_map(&tmX);
        prefetch_map(&tmV);
        for (int s2 = 0; s2 < C::XV_ST; ++s2) {
            mbar_init(&full[s2], 1);
            mbar_init(&empty[s2], kCW);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int64_t ntiles = (N + 63) / 64;
    const int64_t mine = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int nkc = (J + C::XC - 1) / C::XC;
    if (w == kCW) {
        if (lane == 0) {
            int64_t k = 0;
            for (int64_t i = 0; i < mine; ++i) {
                const int r0 = (int)((blockIdx.x + i * gridDim.x) * 64);
                for (int kc = 0; kc < nkc; ++kc, ++k) {
                    const int st = (int)(k % C::XV_ST);
                    if (k >= C::XV_ST) mbar_wait(&empty[st], (uint32_t)(((k / C::XV_ST) - 1) & 1));
                    double *xs = sm + st * C::XV_SD;
                    mbar_arrive_expect_tx(&full[st], (uint32_t)(C::XV_SD * sizeof(double)));
#pragma unroll
                    for (int h2 = 0; h2 < 2; ++h2)
#pragma unroll
                        for (int s = 0; s < 4; ++s)
                            tma_load_2d(xs + (h2 * 4 + s) * 512, &tmX, kc * C::XC + 16 * s, r0 + 32 * h2, &full[st]);
#pragma unroll
                    for (int nv = 0; nv < C::NV; ++nv)
                        tma_load_2d(xs + 4096 + nv * 1024, &tmV, 16 * nv, kc * C::XC, &full[st]);
                }
            }
        }
        return;
    }
    const int wm = w & 3, wn = w >> 2;
    // this lane's two A rows (tile rows 16 wm + 8 i + qperm(g)): box half and row inside the 32-row box
    const int mb0 = 2 * wm, mb1 = 2 * wm + 1;
    const int xo0 = (mb0 >> 2) * 4 * 512, xo1 = (mb1 >> 2) * 4 * 512;
    const int ra0 = 8 * (mb0 & 3) + qperm(g), ra1 = 8 * (mb1 & 3) + qperm(g);
    int64_t k = 0;
    for (int64_t i = 0; i < mine; ++i) {
        double acc[2][NBW][2], acc2[2][NBW][2];  // even / odd columns of a pair: independent chains
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int j = 0; j < NBW; ++j) acc[a][j][0] = acc[a][j][1] = acc2[a][j][0] = acc2[a][j][1] = 0.0;
        for (int kc = 0; kc < nkc; ++kc, ++k) {
            const int st = (int)(k % C::XV_ST);
            mbar_wait(&full[st], (uint32_t)((k / C::XV_ST) & 1));
            const double *xt = sm + st * C::XV_SD;
            const double *vt = xt + 4096;
#pragma unroll
            for (int s = 0; s < 4; ++s)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const double2 a0 = *reinterpret_cast<const double2 *>(xt + xo0 + s * 512 + swz(ra0, 4 * h + t));
                    const double2 a1 = *reinterpret_cast<const double2 *>(xt + xo1 + s * 512 + swz(ra1, 4 * h + t));
                    const int kx = 16 * s + 8 * h + 2 * t;  // chunk column of a.x; a.y is kx + 1
#pragma unroll
                    for (int j = 0; j < NBW; ++j) {
                        const int nb = wn * NBW + j;
                        const int nq = 8 * (nb & 1) + g;  // rank inside the 16-rank box
                        const double *vb = vt + (nb >> 1) * 1024 + (nq & 1);
                        const double bx = vb[swz(kx, nq >> 1)], by = vb[swz(kx + 1, nq >> 1)];
                        dmma884(acc[0][j], a0.x, bx);
                        dmma884(acc2[0][j], a0.y, by);
                        dmma884(acc[1][j], a1.x, bx);
                        dmma884(acc2[1][j], a1.y, by);
                    }
                }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
        }
        const int64_t row0 = (blockIdx.x + i * gridDim.x) * 64;
#pragma unroll
        for (int a = 0; a < 2; ++a) {
            const int64_t grow = row0 + 8 * (2 * wm + a) + qperm(g);
            if (grow < N) {
#pragma unroll
                for (int j = 0; j < NBW; ++j)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int col = 8 * (wn * NBW + j) + 2 * t + e;
                        if (col < R) XV[grow * R + col] = acc[a][j][e] + acc2[a][j][e];
                    }
            }
        }
    }
}

// grid = nJ * nrow CTAs: column block jb = blockIdx.x % nJ (columns FC jb ..), row range
// rs = blockIdx.x / nJ (rows rs * rps .., rps a multiple of 32).  F slot rs gets this block's columns.
template <int RP>
__global__ void __launch_bounds__(kCW * 32 + 32, 1) k_fgemmw(const __grid_constant__ CUtensorMap tmX,
                                                             const __grid_constant__ CUtensorMap tmU, int64_t N, int J,
                                                             int R, int64_t rps, int nJ, double *__restrict__ F_slots,
                                                             double *__restrict__ G_slots) {
    using C = WideCfg<RP>;
    constexpr int NU = C::NV, NR8 = RP / 8, TT = NR8 * NR8;
    extern __shared__ __align__(16) double sm_raw[];
    double *sm = align1k(sm_raw);
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + C::F_ST * C::F_SD);
    uint64_t *empty = full + C::F_ST;
    const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
    const int g = lane >> 2, t = lane & 3;
    if (tid == 0) {
        prefetch_map(&tmX);
        prefetch_map(&tmU);
        for (int s2 = 0; s2 < C::F_ST; ++s2) {
            mbar_init(&full[s2], 1);
            mbar_init(&empty[s2], kCW);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int jb = blockIdx.x % nJ, rs = blockIdx.x / nJ;
    const int j0 = jb * C::FC;
    const int JSa = min(C::FS, (J - j0 + 15) / 16);  // strips of this block that hold real columns
    const int64_t rbeg = (int64_t)rs * rps, rend = min(N, rbeg + rps);
    const int ntl = rbeg < rend ? (int)((rend - rbeg + 31) / 32) : 0;
    if (w == kCW) {
        if (lane == 0) {
            for (int i = 0; i < ntl; ++i) {
                const int st = i % C::F_ST;
                if (i >= C::F_ST) mbar_wait(&empty[st], (uint32_t)(((i / C::F_ST) - 1) & 1));
                double *xs = sm + st * C::F_SD;
                const int r0 = (int)(rbeg + 32 * (int64_t)i);
                mbar_arrive_expect_tx(&full[st], (uint32_t)(JSa + NU) * 4096u);
                for (int s = 0; s < JSa; ++s) tma_load_2d(xs + s * 512, &tmX, j0 + 16 * s, r0, &full[st]);
#pragma unroll
                for (int nu = 0; nu < NU; ++nu) tma_load_2d(xs + (C::FS + nu) * 512, &tmU, 16 * nu, r0, &full[st]);
            }
        }
        return;
    }
    const int pg = qperm(g);
    double acc[C::MAXS][NU][4][2];
#pragma unroll
    for (int q = 0; q < C::MAXS; ++q)
#pragma unroll
        for (int nu = 0; nu < NU; ++nu)
#pragma unroll
            for (int k = 0; k < 4; ++k) acc[q][nu][k][0] = acc[q][nu][k][1] = 0.0;
    // G = US^T US: tile gt = (gi * 8 + w) * nJ + jb of the NR8 x NR8 grid of 8 x 8 tiles
    double gacc[C::GT][2];
#pragma unroll
    for (int gi = 0; gi < C::GT; ++gi) gacc[gi][0] = gacc[gi][1] = 0.0;
    const bool gany = G_slots != nullptr;
    for (int i = 0; i < ntl; ++i) {
        const int st = i % C::F_ST;
        mbar_wait(&full[st], (uint32_t)((i / C::F_ST) & 1));
        const double *xt = sm + st * C::F_SD;
        const double *ut = xt + C::FS * 512;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            const int row = 4 * kk + t;
            if (gany) {
#pragma unroll
                for (int gi = 0; gi < C::GT; ++gi) {
                    const int gt = (gi * kCW + w) * nJ + jb;
                    if (gt < TT) {  // A[m][k] = US[row][8 gm + m], B[k][n] = US[row][8 gn + n]
                        const int ca = 8 * (gt / NR8) + g, cb = 8 * (gt % NR8) + g;
                        dmma884(gacc[gi], ut[(ca >> 4) * 512 + swz(row, (ca & 15) >> 1) + (ca & 1)],
                                ut[(cb >> 4) * 512 + swz(row, (cb & 15) >> 1) + (cb & 1)]);
                    }
                }
            }
            double2 b[NU];
#pragma unroll
            for (int nu = 0; nu < NU; ++nu) b[nu] = *reinterpret_cast<const double2 *>(ut + nu * 512 + swz(row, pg));
#pragma unroll
            for (int q = 0; q < C::MAXS; ++q) {
                const int s = w + kCW * q;
                if (s < JSa) {
                    const double2 a = *reinterpret_cast<const double2 *>(xt + s * 512 + swz(row, pg));
#pragma unroll
                    for (int nu = 0; nu < NU; ++nu) {
                        dmma884(acc[q][nu][0], a.x, b[nu].x);  // even j, even r
                        dmma884(acc[q][nu][1], a.x, b[nu].y);  // even j, odd r
                        dmma884(acc[q][nu][2], a.y, b[nu].x);  // odd j, even r
                        dmma884(acc[q][nu][3], a.y, b[nu].y);  // odd j, odd r
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
    }
    double *slot = F_slots + (int64_t)rs * J * R;
#pragma unroll
    for (int q = 0; q < C::MAXS; ++q) {
        const int s = w + kCW * q;
        if (s < JSa) {
#pragma unroll
            for (int nu = 0; nu < NU; ++nu)
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int j = j0 + 16 * s + 2 * pg + (k >> 1);
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int r = 16 * nu + 2 * qperm(2 * t + e) + (k & 1);
                        if (j < J && r < R) slot[(int64_t)j * R + r] = acc[q][nu][k][e];
                    }
                }
        }
    }
    if (gany) {
        double *gs = G_slots + (int64_t)rs * R * R;
#pragma unroll
        for (int gi = 0; gi < C::GT; ++gi) {
            const int gt = (gi * kCW + w) * nJ + jb;
            if (gt < TT) {
                const int a = 8 * (gt / NR8) + g;
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int b2 = 8 * (gt % NR8) + 2 * t + e;
                    if (a < R && b2 < R) gs[a * R + b2] = gacc[gi][e];
                }
            }
        }
    }
}
