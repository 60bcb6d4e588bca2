// k_slicesw: the per-slice phase for ranks R in (16, 64] (RB = 8 NB = 32 or 64).
//
// Reference: _kernels.py:62-144 (group_update) with the numpy/LU fallback of
// stream.py:319-339 and linalg.py:25-45.  One warp per slice, slices in a
// host-planned order (long slices first), statically strided over the warps of
// a persistent grid (fixed slice -> warp map: deterministic).
//
// Both R x R ridge systems (A = vtv o s s^T + sh I, B = vtv o D_new + sh2 I)
// are factored by a blocked left-looking Cholesky on 8x8 tiles: the tile
// products (the O(R^3) part) run on the FP64 tensor cores (DMMA m8n8k4), the
// 8x8 diagonal blocks are factored and inverted by shuffles.  The data rows
// are solved 8 at a time by blocked forward / backward substitution (again
// DMMA tile products against L and the diagonal inverses); c and the Gram
// U^T U follow from the solved tiles.  The B system's single right-hand side
// rides as row 0 of one 8-row chunk through the same solver.
//
// Shared-memory tiles (8 x 8 doubles) use a swizzle, element (r, c) at
// 8 r + (c ^ 4 ((r >> 1) & 1)), so the three access patterns of the DMMA
// fragments -- A (row l/4, col l%4 + 4h), its transpose, and the accumulator
// pairs (row l/4, cols 2 (l%4) + {0,1}, 16-byte) -- are all bank-conflict free.
//
// G's fresh term sum_k gram_k o w_k w_k^T equals US^T US over all rows
// (US = U o w of the row's slice); the F GEMM forms it (k_fgemm's extra
// column block / k_fgemmw's G tiles), so this kernel writes no G slots.  US
// itself is written by k_us_rows after this kernel (an in-kernel pass cost 4-10x
// more: the warp re-walks its rows behind a 255-register solver).
//
// Failure chain (reference semantics): a non-SPD / non-finite system is
// re-solved by LU with partial pivoting (lane 0, per-warp global scratch);
// an LU zero pivot or a non-finite result reports SolveError for the slice.
// D_old is read once per slice (prefetched into L2 when the slice starts):
// D_new = lam D_old + gram replaces the gram tiles in the warp's scratch, the B
// system, its LU re-solve and the write-back all read it from there.  State
// (W, C, D) is written only after the slice's W solve is validated.
// (included inside dash_update.cu's anonymous namespace)
#pragma once

struct SwParams {
    const int32_t *order;     // batch positions in processing order
    int M;
    const int64_t *row_ptr;
    const int32_t *state_row;
    const uint8_t *is_new;
    const double *XV;         // N x R
    double *U;                // N x R
    double *W, *C, *D;
    const double *vtv;        // R x R
    double *scratch;          // per warp: SwScr<NB>::doubles
    double *vtv_tiles;        // per CTA: NT x 64 doubles
    unsigned long long *err;
    unsigned int *fallbacks;
    int R;
    double lam, eps;
    int pass, final_pass;
};

namespace swk {

__host__ __device__ constexpr int tri(int i, int k) { return i * (i + 1) / 2 + k; }
__device__ __forceinline__ int toff(int r, int c) { return 8 * r + (c ^ ((r & 2) << 1)); }

template <int NB>
struct Cfg {
    static constexpr int RB = 8 * NB;
    static constexpr int NT = NB * (NB + 1) / 2;  // lower tiles
    static constexpr int NW = NB <= 4 ? 16 : 8;   // warps per CTA (one CTA per SM; 8 x 255 registers x 32 = the register file)
    // per warp smem: Lt[NT] | Li[NB] | Uc[NB] | Cs[1] tiles | sv[RB]
    static constexpr int warp_doubles = (NT + 2 * NB + 1) * 64 + RB;
    // vtv's lower tiles live in a per-CTA global scratch (L1-resident, read twice per slice): in shared
    // memory they cost the R = 64 kernel its 8th warp (18 KB against 27.6 KB per warp)
    static constexpr int shared_doubles = 0;
    static constexpr size_t smem_bytes() { return sizeof(double) * (shared_doubles + NW * warp_doubles); }
    // per warp global scratch: GR[NT tiles] | LU matrix RB x RB | row buffer 8 x RB | piv
    static constexpr int scr_doubles = NT * 64 + RB * RB + 8 * RB + RB;
};

struct LaneOff {
    int a0, a1, t0, t1, c;  // A pattern (h = 0, 1), transposed pattern, accumulator pair
    int g, c0;              // accumulator row, first column
};

__device__ __forceinline__ LaneOff lane_offsets() {
    const int l = lane_id(), g = l >> 2, q = l & 3;
    LaneOff o;
    o.a0 = toff(g, q);
    o.a1 = toff(g, q + 4);
    o.t0 = toff(q, g);
    o.t1 = toff(q + 4, g);
    o.c = toff(g, 2 * q);
    o.g = g;
    o.c0 = 2 * q;
    return o;
}

__device__ __forceinline__ void ldc(double (&c)[2], const double *T, const LaneOff &o) {
    const double2 v = *reinterpret_cast<const double2 *>(T + o.c);
    c[0] = v.x;
    c[1] = v.y;
}
__device__ __forceinline__ void stc(double *T, const double (&c)[2], const LaneOff &o) {
    *reinterpret_cast<double2 *>(T + o.c) = make_double2(c[0], c[1]);
}
// c += X Y^T
__device__ __forceinline__ void mma_xyt(double (&c)[2], const double *X, const double *Y, const LaneOff &o) {
    dmma884(c, X[o.a0], Y[o.a0]);
    dmma884(c, X[o.a1], Y[o.a1]);
}
// c -= X Y^T
__device__ __forceinline__ void mma_nxyt(double (&c)[2], const double *X, const double *Y, const LaneOff &o) {
    dmma884(c, -X[o.a0], Y[o.a0]);
    dmma884(c, -X[o.a1], Y[o.a1]);
}
// c += X Y
__device__ __forceinline__ void mma_xy(double (&c)[2], const double *X, const double *Y, const LaneOff &o) {
    dmma884(c, X[o.a0], Y[o.t0]);
    dmma884(c, X[o.a1], Y[o.t1]);
}
// c -= X Y
__device__ __forceinline__ void mma_nxy(double (&c)[2], const double *X, const double *Y, const LaneOff &o) {
    dmma884(c, -X[o.a0], Y[o.t0]);
    dmma884(c, -X[o.a1], Y[o.t1]);
}
// c += X^T Y
__device__ __forceinline__ void mma_xty(double (&c)[2], const double *X, const double *Y, const LaneOff &o) {
    dmma884(c, X[o.t0], Y[o.t0]);
    dmma884(c, X[o.t1], Y[o.t1]);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(FULL_MASK, v, off);
    return v;
}

// Cholesky of the 8x8 SPD diagonal tile T (lower part), right-looking in the
// reference's update order; writes L^{-1} (lower, zeros above) to Li.  Every
// 8-lane group computes the same factor (warp-uniform result).
__device__ __forceinline__ bool diag_chol8(const double *T, double *Li) {
    // Every lane factors the whole tile in registers (36 broadcast loads, ~150 DFMA / DMUL, 8 rsqrt;
    // static indices throughout) and then solves for one column of L^{-1}.  The earlier version kept
    // one row per lane and exchanged pivots and multipliers by shuffles: 33% of the kernel's stall
    // samples and 45% of its instructions at R = 64 (profiles/r02s3_checkpoint/ncu_w64_slicesw_lines.txt).
    const int l = lane_id(), i = l & 7;
    double L[8][8];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int k = 0; k <= r; ++k) L[r][k] = T[toff(r, k)];
    double inv[8];
    bool ok = true;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const double d = L[j][j];
        ok = ok && (d > 0.0) && finite_d(d);
        const double iv = rsqrt_nr(d);  // only 1 / sqrt(d) is needed (L_jj itself is never stored)
        inv[j] = iv;
#pragma unroll
        for (int r = j + 1; r < 8; ++r) L[r][j] *= iv;
#pragma unroll
        for (int k = j + 1; k < 8; ++k)
#pragma unroll
            for (int r = k; r < 8; ++r) L[r][k] = fma(-L[r][j], L[k][j], L[r][k]);
    }
    // column i of L^{-1}:  L x = e_i
    double x[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        double s = (r == i) ? 1.0 : 0.0;
#pragma unroll
        for (int k = 0; k < r; ++k) s = fma(-L[r][k], x[k], s);
        x[r] = s * inv[r];
    }
    if (l < 8) {
#pragma unroll
        for (int r = 0; r < 8; ++r) Li[toff(r, i)] = x[r];
    }
    return ok;
}

// Row-per-lane variant (pivots and multipliers exchanged by shuffles), kept behind -DDASH_DIAG_SHFL
// for A/B.  Same-box A/B at R = 64 (tools/ab_diag.sh, 3 runs each): 3.28-3.33 ms / update with
// this variant, 3.09-3.13 ms with the register-resident factor above; R = 32: slices phase 610 -> 562 us.
__device__ __forceinline__ bool diag_chol8_shfl(const double *T, double *Li) {
    const int l = lane_id(), i = l & 7;
    double row[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) row[k] = (k <= i) ? T[toff(i, k)] : 0.0;
    double inv[8];
    bool ok = true;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const double d = __shfl_sync(FULL_MASK, row[j], j, 8);
        ok = ok && (d > 0.0) && finite_d(d);
        // only 1 / sqrt(d) is needed (L_jj itself is never stored): hardware seed + two
        // Newton steps instead of the IEEE sqrt and two divisions (35% of the kernel's
        // stall samples sat on those three subroutines, profiles/r02s3_w64_ncu.md)
        const double iv = rsqrt_nr(d);
        inv[j] = iv;
        if (i > j) row[j] = row[j] * iv;
#pragma unroll
        for (int k = j + 1; k < 8; ++k) {
            const double lkj = __shfl_sync(FULL_MASK, row[j], k, 8);
            if (i >= k) row[k] = fma(-row[j], lkj, row[k]);
        }
    }
    // column i of L^{-1}:  L x = e_i
    double x[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        double s = (r == i) ? 1.0 : 0.0;
#pragma unroll
        for (int k = 0; k < r; ++k) s = fma(-__shfl_sync(FULL_MASK, row[k], r, 8), x[k], s);
        x[r] = s * inv[r];
    }
    if (l < 8) {
#pragma unroll
        for (int r = 0; r < 8; ++r) Li[toff(r, i)] = x[r];
    }
    return ok;
}

// Blocked left-looking Cholesky of the lower tiles Lt (in place -> L; the
// diagonal tiles keep the updated input, their inverses go to Li).
template <int NB>
__device__ __forceinline__ bool chol_tiles(double *Lt, double *Li, const LaneOff &o) {
    bool ok = true;
#pragma unroll
    for (int jb = 0; jb < NB; ++jb) {
        double c[NB][2];
#pragma unroll
        for (int ib = jb; ib < NB; ++ib) ldc(c[ib], Lt + 64 * tri(ib, jb), o);
        for (int kb = 0; kb < jb; ++kb) {
            const double *Tj = Lt + 64 * tri(jb, kb);
            const double b0 = Tj[o.a0], b1 = Tj[o.a1];
#pragma unroll
            for (int ib = jb; ib < NB; ++ib) {
                const double *Ti = Lt + 64 * tri(ib, kb);
                dmma884(c[ib], -Ti[o.a0], b0);
                dmma884(c[ib], -Ti[o.a1], b1);
            }
        }
#pragma unroll
        for (int ib = jb; ib < NB; ++ib) stc(Lt + 64 * tri(ib, jb), c[ib], o);
        __syncwarp();
#ifdef DASH_DIAG_SHFL  // A/B build knob: the row-per-lane shuffle variant
        constexpr int kSerialMaxNB = 0;
#else
        constexpr int kSerialMaxNB = 8;
#endif
        ok = (NB <= kSerialMaxNB ? diag_chol8(Lt + 64 * tri(jb, jb), Li + 64 * jb)
                      : diag_chol8_shfl(Lt + 64 * tri(jb, jb), Li + 64 * jb)) && ok;
        __syncwarp();
        if (jb + 1 < NB) {
#pragma unroll
            for (int ib = jb + 1; ib < NB; ++ib) {
                c[ib][0] = c[ib][1] = 0.0;
                mma_xyt(c[ib], Lt + 64 * tri(ib, jb), Li + 64 * jb, o);  // L_ib,jb = C L_jj^{-T}
            }
            __syncwarp();
#pragma unroll
            for (int ib = jb + 1; ib < NB; ++ib) stc(Lt + 64 * tri(ib, jb), c[ib], o);
            __syncwarp();
        }
    }
    return ok;
}

// Solve X A^{-1} for an 8-row block X (accumulator layout, in/out), A = L L^T:
// forward Z L^T = X, backward U L = Z.  Leaves the solution tiles in Uc.
template <int NB>
__device__ __forceinline__ void solve_chunk(double (&x)[NB][2], const double *Lt, const double *Li, double *Uc,
                                            double *Cs, const LaneOff &o) {
#pragma unroll
    for (int jb = 0; jb < NB; ++jb) {
        stc(Cs, x[jb], o);
        __syncwarp();
        double z[2] = {0.0, 0.0};
        mma_xyt(z, Cs, Li + 64 * jb, o);
        stc(Uc + 64 * jb, z, o);
        x[jb][0] = z[0];
        x[jb][1] = z[1];
        __syncwarp();
#pragma unroll
        for (int ib = jb + 1; ib < NB; ++ib) mma_nxyt(x[ib], Uc + 64 * jb, Lt + 64 * tri(ib, jb), o);
    }
#pragma unroll
    for (int jb = NB - 1; jb >= 0; --jb) {
        stc(Cs, x[jb], o);
        __syncwarp();
        double u[2] = {0.0, 0.0};
        mma_xy(u, Cs, Li + 64 * jb, o);
        stc(Uc + 64 * jb, u, o);
        x[jb][0] = u[0];
        x[jb][1] = u[1];
        __syncwarp();
#pragma unroll
        for (int ib = 0; ib < jb; ++ib) mma_nxy(x[ib], Uc + 64 * jb, Lt + 64 * tri(jb, ib), o);
    }
}

// LU re-solve of an 8-row block (rare fallback): x staged through Uc, lane i < 8
// solves row i with the LU factors in global scratch.
template <int NB>
__device__ void lu_chunk(double (&x)[NB][2], const double *LUm, const int *piv, double *rowbuf, double *Uc,
                         int R, const LaneOff &o) {
    constexpr int RB = 8 * NB;
#pragma unroll
    for (int jb = 0; jb < NB; ++jb) stc(Uc + 64 * jb, x[jb], o);
    __syncwarp();
    const int l = lane_id();
    if (l < 8) {
        double *rb = rowbuf + l * RB;
        for (int c = 0; c < R; ++c) rb[c] = Uc[64 * (c >> 3) + toff(l, c & 7)];
        lu_solve_serial(LUm, RB, R, piv, rb);
        for (int c = 0; c < R; ++c) Uc[64 * (c >> 3) + toff(l, c & 7)] = rb[c];
    }
    __syncwarp();
#pragma unroll
    for (int jb = 0; jb < NB; ++jb) ldc(x[jb], Uc + 64 * jb, o);
}

}  // namespace swk

template <int NB>
__global__ void __launch_bounds__(swk::Cfg<NB>::NW * 32, 1) k_slicesw(SwParams p) {
    using namespace swk;
    using Cf = Cfg<NB>;
    constexpr int RB = Cf::RB, NT = Cf::NT, NW = Cf::NW;
    extern __shared__ __align__(16) double sm[];
    double *vtvT = p.vtv_tiles + (size_t)blockIdx.x * NT * 64;
    const int w = warp_id(), lane = lane_id();
    double *wb = sm + Cf::shared_doubles + w * Cf::warp_doubles;
    double *Lt = wb, *Li = Lt + 64 * NT, *Uc = Li + 64 * NB, *Cs = Uc + 64 * NB, *sv = Cs + 64;
    const int R = p.R;
    const LaneOff o = lane_offsets();

    // vtv lower tiles (zero padded)
    for (int e = threadIdx.x; e < NT * 64; e += NW * 32) {
        const int t = e >> 6, k = e & 63, r = k >> 3, c = (k & 7) ^ ((r & 2) << 1);
        int ib = 0;
        while (tri(ib + 1, 0) <= t) ++ib;
        const int kb = t - tri(ib, 0);
        const int row = 8 * ib + r, col = 8 * kb + c;
        vtvT[e] = (row < R && col < R) ? p.vtv[row * R + col] : 0.0;
    }
    __syncthreads();

    const int gw = blockIdx.x * NW + w, TW = gridDim.x * NW;
    double *scr = p.scratch + (int64_t)gw * Cf::scr_doubles;
    double *GR = scr, *LUm = GR + 64 * NT, *rowbuf = LUm + RB * RB;
    int *piv = reinterpret_cast<int *>(rowbuf + 8 * RB);

    for (int qi = gw; qi < p.M; qi += TW) {
        const int m = p.order[qi];
        const int64_t r0 = p.row_ptr[m], n = p.row_ptr[m + 1] - r0;
        const int wrow = p.state_row[m];
        const bool fresh = p.is_new[m] != 0;
        const bool boot = fresh && p.pass == 0;
        const double *Dold = p.D + (int64_t)wrow * R * R;
        if (!fresh)  // D_old is needed after the A system and the row solves: start its trip from HBM now
            for (int e = lane * 16; e < R * R; e += 512) asm volatile("prefetch.global.L2 [%0];" ::"l"(Dold + e));
        if (lane * 16 < R) {
            if (!fresh) asm volatile("prefetch.global.L2 [%0];" ::"l"(p.C + (int64_t)wrow * R + lane * 16));
            for (int64_t i = 0; i < (n < 8 ? n : 8); ++i)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(p.XV + (r0 + i) * R + lane * 16));
        }
        __syncwarp();
        for (int r = lane; r < RB; r += 32) sv[r] = r < R ? (boot ? 1.0 : p.W[(int64_t)wrow * R + r]) : 0.0;
        __syncwarp();
        // ---- A = vtv o s s^T + sh I  (_kernels.py:86-97)
        double sh = 0.0;
        for (int r = lane; r < R; r += 32) sh += p.vtv[r * R + r] * sv[r] * sv[r];
        sh = p.eps * warp_sum(sh) / R;
        const int gr = o.g;
#pragma unroll
        for (int ib = 0; ib < NB; ++ib) {
#pragma unroll
            for (int kb = 0; kb <= ib; ++kb) {
                const int t = tri(ib, kb);
                double v[2];
                ldc(v, vtvT + 64 * t, o);
                const int row = 8 * ib + gr;
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int col = 8 * kb + o.c0 + e;
                    double a = v[e] * sv[row] * sv[col];
                    if (row == col) a = row < R ? a + sh : 1.0;
                    v[e] = a;
                }
                stc(Lt + 64 * t, v, o);
            }
        }
        __syncwarp();
        bool okA = chol_tiles<NB>(Lt, Li, o);
        if (!okA) {  // LU on the unpadded system (stream.py:324-329 -> np.linalg.solve)
            if (lane == 0) atomicAdd(p.fallbacks, 1u);
            for (int e = lane; e < R * R; e += 32) {
                const int r = e / R, z = e % R;
                LUm[r * RB + z] = p.vtv[r * R + z] * sv[r] * sv[z] + (r == z ? sh : 0.0);
            }
            __syncwarp();
            int okf = 1;
            if (lane == 0) okf = lu_factor_serial(LUm, RB, R, piv) ? 1 : 0;
            okf = __shfl_sync(FULL_MASK, okf, 0);
            if (!okf && lane == 0) report_error(p.err, m, DASH_E_SINGULAR);
            __syncwarp();
        }
        // ---- rows: U, c partials, gram into GR (8 rows per chunk)
        double cp[NB][2];
#pragma unroll
        for (int jb = 0; jb < NB; ++jb) cp[jb][0] = cp[jb][1] = 0.0;
        const int nch = (int)((n + 7) >> 3);
        for (int ch = 0; ch < nch; ++ch) {
            const int64_t ri = (int64_t)ch * 8 + gr;
            const bool valid = ri < n;
            const double *xrow = p.XV + (r0 + ri) * R;
            double xr[NB][2], x[NB][2];
#pragma unroll
            for (int jb = 0; jb < NB; ++jb)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int col = 8 * jb + o.c0 + e;
                    const double v = (valid && col < R) ? xrow[col] : 0.0;
                    xr[jb][e] = v;
                    x[jb][e] = v * sv[col];
                }
            __syncwarp();  // previous chunk's reads of Uc are done
            if (okA) solve_chunk<NB>(x, Lt, Li, Uc, Cs, o);
            else lu_chunk<NB>(x, LUm, piv, rowbuf, Uc, R, o);
            double *urow = p.U + (r0 + ri) * R;
#pragma unroll
            for (int jb = 0; jb < NB; ++jb)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int col = 8 * jb + o.c0 + e;
                    if (valid && col < R) urow[col] = x[jb][e];
                    cp[jb][e] = fma(xr[jb][e], x[jb][e], cp[jb][e]);
                }
            __syncwarp();
#pragma unroll
            for (int ib = 0; ib < NB; ++ib)
#pragma unroll
                for (int kb = 0; kb <= ib; ++kb) {
                    const int t = tri(ib, kb);
                    double gacc[2] = {0.0, 0.0};
                    if (ch > 0) ldc(gacc, GR + 64 * t, o);
                    mma_xty(gacc, Uc + 64 * ib, Uc + 64 * kb, o);
                    stc(GR + 64 * t, gacc, o);
                }
        }
        if (nch == 0) {
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const double z[2] = {0.0, 0.0};
                stc(GR + 64 * t, z, o);
            }
        }
        // c = lam c_old + sum_i xv o u  (rows reduced across the 8 lane rows)
#pragma unroll
        for (int jb = 0; jb < NB; ++jb)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                double v = cp[jb][e];
                v += __shfl_xor_sync(FULL_MASK, v, 4);
                v += __shfl_xor_sync(FULL_MASK, v, 8);
                v += __shfl_xor_sync(FULL_MASK, v, 16);
                const int col = 8 * jb + o.c0 + e;
                cp[jb][e] = col < R ? p.lam * (fresh ? 0.0 : p.C[(int64_t)wrow * R + col]) + v : 0.0;
            }
        // ---- B = vtv o D_new + sh2 I, D_new = lam D_old + gram  (_kernels.py:103-128)
        __syncwarp();
        double sh2 = 0.0;
        {
            double bd[NB][2];
#pragma unroll
            for (int jb = 0; jb < NB; ++jb) {
                const int t = tri(jb, jb);
                double g2[2], v[2];
                ldc(g2, GR + 64 * t, o);
                ldc(v, vtvT + 64 * t, o);
                const int row = 8 * jb + gr;
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int col = 8 * jb + o.c0 + e;
                    const int rr = row >= col ? row : col, cc = row >= col ? col : row;  // lower element
                    double dn = 0.0;
                    if (row < R && col < R) dn = p.lam * (fresh ? 0.0 : Dold[rr * R + cc]) + g2[e];
                    g2[e] = dn;
                    bd[jb][e] = v[e] * dn;
                    if (row == col && row < R) sh2 += v[e] * dn;
                }
                stc(GR + 64 * t, g2, o);  // GR now holds D_new (D_old is read exactly once per slice)
            }
            sh2 = p.eps * warp_sum(sh2) / R;
#pragma unroll
            for (int jb = 0; jb < NB; ++jb) {
                const int row = 8 * jb + gr;
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int col = 8 * jb + o.c0 + e;
                    if (row == col) bd[jb][e] = row < R ? bd[jb][e] + sh2 : 1.0;
                }
                stc(Lt + 64 * tri(jb, jb), bd[jb], o);
            }
        }
#pragma unroll
        for (int ib = 1; ib < NB; ++ib) {
            // the block row's D_old pairs first (independent loads in flight together; the
            // stores below would otherwise fence each tile's loads behind the previous tile)
            const int row = 8 * ib + gr;
            double dd[NB - 1][2];
#pragma unroll
            for (int kb = 0; kb < ib; ++kb) {
                const int col = 8 * kb + o.c0;  // even; R even -> 16-byte aligned pair
                double2 d2 = make_double2(0.0, 0.0);
                if (!fresh && row < R && col + 1 < R) d2 = __ldcg(reinterpret_cast<const double2 *>(Dold + row * R + col));
                else if (!fresh && row < R && col < R) d2.x = __ldcg(Dold + row * R + col);
                dd[kb][0] = d2.x;
                dd[kb][1] = d2.y;
            }
#pragma unroll
            for (int kb = 0; kb < ib; ++kb) {
                const int t = tri(ib, kb);
                double g2[2], v[2];
                ldc(g2, GR + 64 * t, o);
                ldc(v, vtvT + 64 * t, o);
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int col = 8 * kb + o.c0 + e;
                    double dn = 0.0;
                    if (row < R && col < R) dn = p.lam * dd[kb][e] + g2[e];
                    g2[e] = dn;
                    v[e] *= dn;
                }
                stc(GR + 64 * t, g2, o);
                stc(Lt + 64 * t, v, o);
            }
        }
        __syncwarp();
        const bool okB = chol_tiles<NB>(Lt, Li, o);
        double wv[NB][2];
#pragma unroll
        for (int jb = 0; jb < NB; ++jb)
#pragma unroll
            for (int e = 0; e < 2; ++e) wv[jb][e] = gr == 0 ? cp[jb][e] : 0.0;
        if (okB) solve_chunk<NB>(wv, Lt, Li, Uc, Cs, o);
        bool fin = true;
#pragma unroll
        for (int jb = 0; jb < NB; ++jb)
#pragma unroll
            for (int e = 0; e < 2; ++e) fin = fin && finite_d(wv[jb][e]);
        if (!(okB && __all_sync(FULL_MASK, fin))) {
            // LU on the unpadded B system from the D_new tiles in GR
            if (lane == 0) atomicAdd(p.fallbacks, 1u);
            double shb = 0.0;
            for (int r = lane; r < R; r += 32)
                shb += p.vtv[r * R + r] * GR[64 * tri(r >> 3, r >> 3) + toff(r & 7, r & 7)];
            shb = p.eps * warp_sum(shb) / R;
            for (int e = lane; e < R * R; e += 32) {
                const int r = e / R, z = e % R;
                const int rr = r >= z ? r : z, cc = r >= z ? z : r;
                const double dn = GR[64 * tri(rr >> 3, cc >> 3) + toff(rr & 7, cc & 7)];
                LUm[r * RB + z] = p.vtv[r * R + z] * dn + (r == z ? shb : 0.0);
            }
            __syncwarp();
            int okf = 1;
            if (lane == 0) okf = lu_factor_serial(LUm, RB, R, piv) ? 1 : 0;
            okf = __shfl_sync(FULL_MASK, okf, 0);
            if (!okf && lane == 0) report_error(p.err, m, DASH_E_SINGULAR);
#pragma unroll
            for (int jb = 0; jb < NB; ++jb)
#pragma unroll
                for (int e = 0; e < 2; ++e) wv[jb][e] = gr == 0 ? cp[jb][e] : 0.0;
            lu_chunk<NB>(wv, LUm, piv, rowbuf, Uc, R, o);
            fin = true;
#pragma unroll
            for (int jb = 0; jb < NB; ++jb)
#pragma unroll
                for (int e = 0; e < 2; ++e) fin = fin && finite_d(wv[jb][e]);
            if (!__all_sync(FULL_MASK, fin) && lane == 0) report_error(p.err, m, DASH_E_NONFINITE);
        }
        // ---- write-back: W (every pass), C and D (final pass)
        if (gr == 0) {
#pragma unroll
            for (int jb = 0; jb < NB; ++jb)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int col = 8 * jb + o.c0 + e;
                    if (col < R) {
                        p.W[(int64_t)wrow * R + col] = wv[jb][e];
                        if (p.final_pass) p.C[(int64_t)wrow * R + col] = cp[jb][e];
                    }
                }
        }
        if (p.final_pass) {
            double *Dn = p.D + (int64_t)wrow * R * R;
            // D_new from GR (each lane reads back the pairs it stored itself)
#pragma unroll
            for (int ib = 0; ib < NB; ++ib)
#pragma unroll
                for (int kb = 0; kb <= ib; ++kb) {
                    const int t = tri(ib, kb);
                    double g2[2];
                    ldc(g2, GR + 64 * t, o);
                    const int row = 8 * ib + gr;
                    if (ib == kb) {  // diagonal tile: GR holds it fully symmetric
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int col = 8 * kb + o.c0 + e;
                            if (row < R && col < R) Dn[row * R + col] = g2[e];
                        }
                    } else {  // lower tile rows, then its transpose (through Cs) as rows of the upper tile
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int col = 8 * kb + o.c0 + e;
                            if (row < R && col < R) Dn[row * R + col] = g2[e];
                        }
                        __syncwarp();
                        stc(Cs, g2, o);
                        __syncwarp();
                        const int urow = 8 * kb + gr;
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int ucol = 8 * ib + o.c0 + e;
                            if (urow < R && ucol < R) Dn[urow * R + ucol] = Cs[toff(o.c0 + e, gr)];
                        }
                    }
                }
        }
    }
}
