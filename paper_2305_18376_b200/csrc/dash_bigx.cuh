// Fused big-slice path (R bucket 16, FP64, TMA): the rows of BIG slices
// (> kSmallRows rows) are read from HBM ONCE.  The old path read them three
// times (X in the XV GEMM, XV in k_big, X again in the F GEMM) plus wrote and
// re-read XV / U o w.  Here, per 32-row tile of a big slice:
//
//   XV   = X V                   (DMMA, X as swizzled TMA boxes)
//   U    = XV Ms^T               (DMMA; Ms = A^{-1} diag(s) of the slice)  -> U_out
//   c   += diag(XV^T U)          (fragment FMAs)
//   gram+= U^T U                 (DMMA)
//   P   += X^T U                 (DMMA, J x R, X still in shared memory)
//
// and the slice's F contribution X^T (U o w) = P diag(w) is formed once w is
// known (stream.py:321; only the row-sum order differs).  Three kernels:
//
//   k_bigx_pre   one warp per big slice: the A system by the symmetric sweep
//                (LU fallback) -> Ms (global); zeroes U o w on the slice's
//                partial boundary tiles (the small-row F GEMM may read those
//                tiles); block 0 scans the slices' tile counts -> toff[].
//   k_bigx       persistent, one CTA per SM, warp-specialised (producer warp,
//                4 XV / U warps, 4 X^T U / gram warps, mbarrier handoffs, no
//                CTA barriers in the loop): the big slices' tiles, in plan
//                order, are split EVENLY over the CTAs (a slice may span CTAs);
//                each (slice, CTA) segment writes its partial P, gram, c to
//                parts[slice + CTA] (unique: slices and CTAs are both ordered).
//   k_bigx_post  one CTA per big slice: segment partials summed in CTA order
//                (deterministic), D = lam D + gram, the S-row system (Gauss-
//                Jordan, LU fallback) -> w; W / C / D rows; G slot gram o w w^T;
//                F slot P diag(w).
//
// (included inside dash_update.cu's anonymous namespace, after dash_big.cuh)
#pragma once

constexpr int kBxRB = 16;           // rank bucket
constexpr int kBxMP = kBxRB + 4;    // Ms pitch (B-frag reads)
constexpr int kBxUP = kBxRB + 8;    // U tile pitch (gram frags conflict-free)

constexpr int kBxMaxStages = 6;
#ifndef DASH_BXA
#define DASH_BXA 8
#endif
#ifndef DASH_BXB
#define DASH_BXB 4
#endif
constexpr int kBxA = DASH_BXA;                    // XV / U warps: kBxA / 4 tiles in flight (4 row blocks each)
constexpr int kBxB = DASH_BXB;                    // X^T U / gram warps: P strips b, b + kBxB, ... (J <= 128)
constexpr int kBxThreads = (kBxA + kBxB + 1) * 32;  // + the producer warp
constexpr int kBxUSlots = 4;                      // U hand-off buffers
// Shared-memory plan of k_bigx for X in FP64 (boxes of 16 doubles x 32 rows)
// or FP32 (the FP32 data mode: boxes of 32 floats x 32 rows).  A box is 4 KB
// either way (32 rows of one 128-byte swizzled line).
template <typename TX>
struct BigxSmemT {
    static constexpr bool F32 = sizeof(TX) == 4;
    static constexpr int CW = F32 ? 32 : 16;  // X columns per box
    static __host__ __device__ int strips(int J) { return (J + CW - 1) / CW; }
    static __host__ __device__ int stages(int J) { return F32 ? (strips(J) <= 4 ? 6 : 3) : (strips(J) <= 8 ? 4 : 2); }
    // V^T pitch: == 8 (mod 16) doubles for the FP64 fragment pairs, == 2 (mod 16) for the FP32 quads
    static __host__ __device__ int vtp(int J) { return strips(J) * CW + (F32 ? 2 : 8); }
    static __host__ __device__ size_t stage_doubles(int J) { return (size_t)strips(J) * 512; }
    // [stages x JS boxes] | vt[16 x VTP] | ubuf[kBxUSlots][32 x 16 swz] | barriers
    static __host__ __device__ size_t bytes(int J) {
        return 1024 + sizeof(double) * (stages(J) * stage_doubles(J) + 16 * (size_t)vtp(J) + 512 * kBxUSlots) +
               8 * (2 * kBxMaxStages + 2 * kBxUSlots);
    }
    // partial slot of one (slice, CTA) segment: P[J x 16] | gram[16 x 16] | c[kBxA][16]
    static __host__ __device__ int64_t part_doubles(int J) { return (int64_t)J * 16 + 256 + 16 * kBxA; }
};
using BigxSmem = BigxSmemT<double>;

// element (row, col) of a 32 x 16 swizzled double tile (16-byte chunk c at c ^ (row & 7))
__device__ __forceinline__ int swz_e(int row, int col) { return swz(row, col >> 1) + (col & 1); }

// CTA c of G owns tiles [tile_start(c), tile_start(c + 1)) of the T big-slice tiles
__host__ __device__ __forceinline__ int64_t tile_start(int64_t c, int64_t T, int64_t G) {
    const int64_t base = T / G, rem = T % G;
    return c * base + (c < rem ? c : rem);
}
__device__ __forceinline__ int64_t cta_of_tile(int64_t tau, int64_t T, int64_t G) {
    const int64_t base = T / G, rem = T % G;
    const int64_t split = rem * (base + 1);
    return tau < split ? tau / (base + 1) : rem + (tau - split) / base;
}

struct BigxParams {
    const int4 *meta;         // device plan: big slice bi at meta[nsmall + bi]
    const int *plan_counts;   // {nsmall, nbig}
    const double *V;          // J x R
    const double *vtv;        // R x R (written by the XV kernel)
    const double *W, *C;      // state (read)
    double *Wo, *Co, *D;      // state (written by post)
    double *U, *US;           // U_out; U o w workspace (boundary rows zeroed)
    double *ms;               // nbig x 16 x kBxMP: Ms per big slice
    int *toff;                // nbig + 1: tile offsets in plan order
    double *parts;            // (nbig + G) x part_doubles
    double *F_slots;          // post: one J x R slot per big slice
    double *G_slots;          // post: one R x R slot per big slice
    unsigned long long *err;
    unsigned int *fallbacks;
    int64_t N, T;             // rows in the batch; big-slice tiles
    int J, R, G;              // G = k_bigx grid
    double lam, eps;
    int pass, final_pass;
    int post_wait;            // k_bigx_post: wait for k_bigx up front (no F GEMM between them)
};

// ---------------------------------------------------------------------------
// k_bigx_pre: block 0 = tile scan; blocks >= 1: one warp per big slice (A system)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_bigx_pre(BigxParams p) {
    constexpr int RB = kBxRB, LDV = RB + 2, LDL = RB + 1;
    __shared__ double vtv_s[RB * LDV];
    __shared__ __align__(16) double wbuf[8][2 * RB + RB * LDL + RB];  // gather bufs (2) | lu | s
    __shared__ int wpiv[8][RB];
    // launched behind the small-slice kernel, which triggered only after its
    // own pdl_wait: the XV kernel's vtv and the plan are complete and visible.
    // No early trigger: the streaming kernel behind this one must not become
    // resident (150 KB of shared memory per SM) while small slices still run.
    const int lane = lane_id(), w = warp_id();
    const int nsmall = __ldcg(p.plan_counts), nbig = __ldcg(p.plan_counts + 1);
    const int R = p.R;
    if (blockIdx.x == 0) {
        if (w == 0) {  // toff = exclusive scan of ceil(n / 32) in plan order
            int run = 0;
            for (int b0 = 0; b0 < nbig; b0 += 32) {
                const int bi = b0 + lane;
                const int nt = bi < nbig ? (int)((__ldcg(&p.meta[nsmall + bi].y) + kTR - 1) / kTR) : 0;
                int inc = nt;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const int u = __shfl_up_sync(FULL_MASK, inc, d);
                    if (lane >= d) inc += u;
                }
                if (bi < nbig) p.toff[bi] = run + inc - nt;
                run += __shfl_sync(FULL_MASK, inc, 31);
            }
            if (lane == 0) p.toff[nbig] = run;
        }
        pdl_wait();
        pdl_trigger();
        return;
    }
    for (int i = threadIdx.x; i < RB * LDV; i += blockDim.x) {
        const int a = i / LDV, b = i % LDV;
        vtv_s[i] = (a < R && b < R) ? __ldcg(p.vtv + a * R + b) : 0.0;
    }
    __syncthreads();
    const int bi = (blockIdx.x - 1) * 8 + w;
    if (bi < nbig) {
        const int4 mt = __ldcg(p.meta + nsmall + bi);
        const int m = mt.w;
        const int64_t r0 = mt.x, n = mt.y;
        const int wrow = mt.z & 0x7fffffff;
        const bool fresh = mt.z < 0;
        double *buf = wbuf[w];
        double *lu = buf + 2 * RB;
        double *svec = lu + RB * LDL;
        const int r = lane % RB;
        const bool real = lane < RB && r < R;
        if (lane < RB) svec[lane] = real ? ((fresh && p.pass == 0) ? 1.0 : __ldcg(p.W + (int64_t)wrow * R + r)) : 0.0;
        __syncwarp();
        const double s_r = real ? svec[r] : 0.0;
        double sh = 0.0;
#pragma unroll
        for (int z = 0; z < RB; ++z)
            if (z < R) sh += vtv_s[z * LDV + z] * svec[z] * svec[z];
        sh = p.eps * sh / R;
        const double dg = real ? sh : 1.0;
        const double *vrow = vtv_s + r * LDV;
        double a2[RB];
#pragma unroll
        for (int z = 0; z < RB; ++z) a2[z] = (lane < RB ? vrow[z] * s_r * svec[z] : 0.0) + ((z == r) ? dg : 0.0);
        // lanes 0..15 sweep A; lanes 16..31 sweep a harmless identity (own gather buffer)
        const bool okA = sweep_inverse<RB>(a2, lane < RB ? buf : buf + RB, r);
        const unsigned badA = __ballot_sync(FULL_MASK, !okA) & 0xffffu;
        if (badA) {
            const bool need = lane < RB;
#pragma unroll
            for (int z = 0; z < RB; ++z)
                if (need) a2[z] = vrow[z] * s_r * svec[z] + ((z == r) ? dg : 0.0);
            if (lane == 0) atomicAdd(p.fallbacks, 1u);
            const bool okLU = lu_fallback<RB>(a2, lu, wpiv[w], r, R, need);
            if (lane == 0 && !okLU) report_error(p.err, m, DASH_E_SINGULAR);
        }
        // Ms[n][k] = A^{-1}[n][k] s_k  (a2 holds -A^{-1}), so U = XV Ms^T
        if (lane < RB) {
            double *msr = p.ms + (int64_t)bi * RB * kBxMP + r * kBxMP;
#pragma unroll
            for (int z = 0; z < RB; ++z) msr[z] = (r < R && z < R) ? -a2[z] * svec[z] : 0.0;
        }
        // U o w rows of the partial boundary tiles (the small-row F GEMM may read them)
        if (p.US != nullptr) {
            const int64_t e0 = min(r0 + n, (r0 + kTR - 1) / kTR * kTR);  // end of the first partial tile
            const int64_t s1 = max(e0, (r0 + n) / kTR * kTR);            // start of the last partial tile
            for (int64_t row = r0 + lane / R; row < e0; row += 32 / R)
                if (lane < (32 / R) * R) p.US[row * R + lane % R] = 0.0;
            for (int64_t row = s1 + lane / R; row < r0 + n; row += 32 / R)
                if (lane < (32 / R) * R) p.US[row * R + lane % R] = 0.0;
        }
    }
    pdl_wait();  // completion of this grid implies completion of the small-slice kernel
    pdl_trigger();
}

// ---------------------------------------------------------------------------
// k_bigx: the streaming fused kernel.  Warp-specialised, no CTA barriers in
// the tile loop:
//   producer warp     TMA ring of 32-row X tiles (JS swizzled 16-column boxes)
//   group A (warps 0-3, warp = 8-row block mb of the tile):
//                     XV = X V (DMMA, 4 chains), U = XV Ms^T straight from the
//                     XV accumulator fragments (the K order of the U product
//                     is permuted to the C-fragment layout: no shuffles), c
//                     partial, U -> U_out and -> ubuf[tile & 1]
//   group B (warps 4-7, warp b = strips s == b (mod 4) of P, gram tile b):
//                     P += X^T U (DMMA, X still in the stage), gram += U^T U
// A runs up to two tiles ahead of B (ubuf double-buffered, uready / ufree
// mbarriers); a stage is released when both groups are done with it.
// Partials of (slice, CTA): A writes c, B writes P and gram (disjoint parts).
// ---------------------------------------------------------------------------
template <int MAXS, int JSC, typename TX>
__global__ void __maxnreg__(128) k_bigx(const __grid_constant__ CUtensorMap tmX, BigxParams p) {
    using SM = BigxSmemT<TX>;
    constexpr bool F32 = SM::F32;
    extern __shared__ __align__(16) double sm_raw[];
    double *sm = align1k(sm_raw);
    const int J = p.J, R = p.R;
    const int JS = JSC ? JSC : SM::strips(J), VTP = SM::vtp(J), NST = SM::stages(J);
    const size_t SD = SM::stage_doubles(J);
    double *xs = sm;
    double *vt = xs + NST * SD;          // vt[n][k] = V[k][n]
    double *ubuf = vt + 16 * VTP;        // kBxUSlots x (32 x 16 swizzled)
    uint64_t *full = reinterpret_cast<uint64_t *>(ubuf + 512 * kBxUSlots);
    uint64_t *empty = full + kBxMaxStages;
    uint64_t *uready = empty + kBxMaxStages;
    uint64_t *ufree = uready + kBxUSlots;
    const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
    const int g = lane >> 2, t = lane & 3;
    pdl_wait();  // Ms, toff from k_bigx_pre (and, transitively, XV / plan / small slices)
    pdl_trigger();
    if (tid == 0) {
        prefetch_map(&tmX);
        for (int s2 = 0; s2 < NST; ++s2) {
            mbar_init(&full[s2], 1);
            mbar_init(&empty[s2], 4 + kBxB);  // the 4 XV warps of the tile's parity + every X^T U warp
        }
        for (int b = 0; b < kBxUSlots; ++b) {
            mbar_init(&uready[b], 4);
            mbar_init(&ufree[b], kBxB);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int nsmall = __ldcg(p.plan_counts);
    const int64_t T = p.T, G = p.G;
    const int64_t tau0 = tile_start(blockIdx.x, T, G), tau1 = tile_start(blockIdx.x + 1, T, G);
    if (tau0 >= tau1) return;
    int bi0 = 0;  // first big slice of this CTA's range: last bi with toff[bi] <= tau0
    {
        const int nbig = __ldcg(p.plan_counts + 1);
        int lo = 0, hi = nbig - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (__ldcg(p.toff + mid) <= tau0) lo = mid;
            else hi = mid - 1;
        }
        bi0 = lo;
    }
    // slice tracking shared by every role: advance to the slice of tile tau
    int bi = bi0 - 1;
    int64_t tb = 0, te = 0, r0 = 0, n = 0;
    auto advance = [&](int64_t tau) -> bool {
        if (tau < te) return false;
        do {
            ++bi;
            tb = __ldcg(p.toff + bi);
            te = __ldcg(p.toff + bi + 1);
        } while (tau >= te);
        const int4 mt = __ldcg(p.meta + nsmall + bi);
        r0 = mt.x;
        n = mt.y;
        return true;
    };
    const int64_t PD = BigxSmem::part_doubles(J);
    if (w == kBxA + kBxB) {  // ---------------- producer
        if (lane == 0) {
            for (int64_t tau = tau0, i = 0; tau < tau1; ++tau, ++i) {
                advance(tau);
                const int st = (int)(i % NST);
                if (i >= NST) mbar_wait(&empty[st], (uint32_t)(((i / NST) - 1) & 1));
                const int row0 = (int)(r0 + (tau - tb) * kTR);
                mbar_arrive_expect_tx(&full[st], (uint32_t)JS * 4096u);
                for (int s = 0; s < JS; ++s) tma_load_2d(xs + st * SD + s * 512, &tmX, SM::CW * s, row0, &full[st]);
            }
        }
        return;
    }
    if (w < kBxA) {  // ---------------- group A: XV, U, c; tiles of parity w / 4, rows 8 mb .. 8 mb + 7
        for (int i = tid; i < 16 * VTP; i += kBxA * 32) {  // V^T staging overlaps the producer's first loads
            const int nn = i / VTP, k = i % VTP;
            vt[i] = (nn < R && k < J) ? p.V[k * R + nn] : 0.0;
        }
        asm volatile("bar.sync 2, %0;" ::"n"(kBxA * 32) : "memory");  // the XV warps only
        const int par = w >> 2, mb = w & 3;
        constexpr int NPAR = kBxA / 4;  // tiles in flight on the XV side
        const int xrow = 8 * mb + qperm(g);  // A-fragment / output row (conflict-free X reads)
        double msf[4][2];                    // B frags of U = XV Ms^T in the permuted K order
        int msf_bi = -1;
        double cacc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
        for (int64_t tau = tau0, i = 0; tau < tau1; ++tau, ++i) {
            advance(tau);
            if ((int)(i % NPAR) == par) {
                if (msf_bi != bi) {
                    // K step kk feeds XV column col(kk, t) = 8 (kk >> 1) + 2 t + (kk & 1) (the C layout)
                    const double *msg = p.ms + (int64_t)bi * 16 * kBxMP;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
#pragma unroll
                        for (int nb = 0; nb < 2; ++nb)
                            msf[kk][nb] = __ldcg(msg + (8 * nb + g) * kBxMP + 8 * (kk >> 1) + 2 * t + (kk & 1));
                    msf_bi = bi;
                }
                const int64_t row0 = r0 + (tau - tb) * kTR;
                const int nvalid = (int)min((int64_t)kTR, r0 + n - row0);
                const int st = (int)(i % NST);
                mbar_wait(&full[st], (uint32_t)((i / NST) & 1));
                const double *xt = xs + st * SD;
                double xa[2][4][2];  // [nb][K chain][2]
    #pragma unroll
                for (int nb = 0; nb < 2; ++nb)
    #pragma unroll
                    for (int c = 0; c < 4; ++c) xa[nb][c][0] = xa[nb][c][1] = 0.0;
                if constexpr (!F32) {
    #pragma unroll
                    for (int s = 0; s < JS; ++s) {
    #pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const double2 a = *reinterpret_cast<const double2 *>(xt + s * 512 + swz(xrow, 4 * h + t));
    #pragma unroll
                            for (int nb = 0; nb < 2; ++nb) {
                                const double2 b =
                                    *reinterpret_cast<const double2 *>(vt + (8 * nb + g) * VTP + 16 * s + 8 * h + 2 * t);
                                dmma884(xa[nb][2 * h], a.x, b.x);
                                dmma884(xa[nb][2 * h + 1], a.y, b.y);
                            }
                        }
                    }
                } else {  // FP32 boxes: one float4 = 4 consecutive columns 32 s + 16 h + 4 t + {0..3}
                    const float *xf = reinterpret_cast<const float *>(xt);
    #pragma unroll
                    for (int s = 0; s < JS; ++s) {
    #pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const float4 a = *reinterpret_cast<const float4 *>(xf + s * 1024 + swzf(xrow, 4 * h + t));
    #pragma unroll
                            for (int nb = 0; nb < 2; ++nb) {
                                const double *vb = vt + (8 * nb + g) * VTP + 32 * s + 16 * h + 4 * t;
                                const double2 b0 = *reinterpret_cast<const double2 *>(vb);
                                const double2 b1 = *reinterpret_cast<const double2 *>(vb + 2);
                                dmma884(xa[nb][0], (double)a.x, b0.x);
                                dmma884(xa[nb][1], (double)a.y, b0.y);
                                dmma884(xa[nb][2], (double)a.z, b1.x);
                                dmma884(xa[nb][3], (double)a.w, b1.y);
                            }
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[st]);
                const bool ok = xrow < nvalid;
                double xv[2][2];
#pragma unroll
                for (int nb = 0; nb < 2; ++nb)
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        xv[nb][e] = ok ? (xa[nb][0][e] + xa[nb][1][e]) + (xa[nb][2][e] + xa[nb][3][e]) : 0.0;
                // U = XV Ms^T: A fragment of K step kk = this lane's XV value xv[kk >> 1][kk & 1]
                double ua[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
#pragma unroll
                    for (int nb = 0; nb < 2; ++nb) dmma884(ua[nb], xv[kk >> 1][kk & 1], msf[kk][nb]);
                const int bsel = (int)(i % kBxUSlots);
                if (i >= kBxUSlots) mbar_wait(&ufree[bsel], (uint32_t)(((i / kBxUSlots) - 1) & 1));
                double *ub = ubuf + bsel * 512;
#pragma unroll
                for (int nb = 0; nb < 2; ++nb) {
                    const int col = 8 * nb + 2 * t;
                    cacc[nb][0] = fma(xv[nb][0], ua[nb][0], cacc[nb][0]);
                    cacc[nb][1] = fma(xv[nb][1], ua[nb][1], cacc[nb][1]);
                    *reinterpret_cast<double2 *>(ub + swz_e(xrow, col)) = make_double2(ua[nb][0], ua[nb][1]);
                    if (ok && col < R)
                        *reinterpret_cast<double2 *>(p.U + (row0 + xrow) * R + col) = make_double2(ua[nb][0], ua[nb][1]);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&uready[bsel]);
            }
            if (tau == te - 1 || tau == tau1 - 1) {  // c partial of (slice, CTA): this warp's tiles
                double *cp = p.parts + (int64_t)(bi + blockIdx.x) * PD + (int64_t)J * 16 + 256 + w * 16;
#pragma unroll
                for (int nb = 0; nb < 2; ++nb)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        double v = cacc[nb][e];
                        v += __shfl_xor_sync(FULL_MASK, v, 4);
                        v += __shfl_xor_sync(FULL_MASK, v, 8);
                        v += __shfl_xor_sync(FULL_MASK, v, 16);
                        if (g == 0) cp[8 * nb + 2 * t + e] = v;
                        cacc[nb][e] = 0.0;
                    }
            }
        }
        return;
    }
    // ---------------- group B: P += X^T U (strips b, b + 8, ...), gram tile b (b < 4)
    const int b = w - kBxA;
    const int pg = qperm(g);
    const int mi = (b >> 1) & 1, ni = b & 1;
    // FP64: pacc[q][k] = (j parity k >> 1, r parity k & 1) of strip q's 2x2 block;
    // FP32: pacc[q][2 e + f] = (j = 4 pg + e, r parity f) of strip q's 4x2 block
    constexpr int NPT = F32 ? 8 : 4;
    double pacc[MAXS][NPT][2];
    double gacc[2] = {0.0, 0.0};
#pragma unroll
    for (int q = 0; q < MAXS; ++q)
#pragma unroll
        for (int k = 0; k < NPT; ++k) pacc[q][k][0] = pacc[q][k][1] = 0.0;
    for (int64_t tau = tau0, i = 0; tau < tau1; ++tau, ++i) {
        advance(tau);
        const int st = (int)(i % NST);
        const int bsel = (int)(i % kBxUSlots);
        mbar_wait(&uready[bsel], (uint32_t)((i / kBxUSlots) & 1));
        mbar_wait(&full[st], (uint32_t)((i / NST) & 1));  // completed long ago (group A waited on it)
        const double *xt = xs + st * SD;
        const double *ub = ubuf + bsel * 512;
#pragma unroll
        for (int kk = 0; kk < kTR / 4; ++kk) {
            const int row = 4 * kk + t;
            const double2 bu = *reinterpret_cast<const double2 *>(ub + swz(row, pg));  // U[row][2pg, 2pg+1]
#pragma unroll
            for (int q = 0; q < MAXS; ++q) {
                const int s = b + kBxB * q;
                if (s < JS) {
                    if constexpr (!F32) {
                        const double2 a = *reinterpret_cast<const double2 *>(xt + s * 512 + swz(row, pg));
                        dmma884(pacc[q][0], a.x, bu.x);
                        dmma884(pacc[q][1], a.x, bu.y);
                        dmma884(pacc[q][2], a.y, bu.x);
                        dmma884(pacc[q][3], a.y, bu.y);
                    } else {
                        const float4 a = *reinterpret_cast<const float4 *>(reinterpret_cast<const float *>(xt) +
                                                                           s * 1024 + swzf(row, pg));
                        const double av[4] = {(double)a.x, (double)a.y, (double)a.z, (double)a.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            dmma884(pacc[q][2 * e], av[e], bu.x);
                            dmma884(pacc[q][2 * e + 1], av[e], bu.y);
                        }
                    }
                }
            }
            if (b < 4) dmma884(gacc, ub[swz_e(row, 8 * mi + g)], ub[swz_e(row, 8 * ni + g)]);
        }
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(&empty[st]);
            mbar_arrive(&ufree[bsel]);
        }
        if (tau == te - 1 || tau == tau1 - 1) {  // P strips and gram tile of (slice, CTA)
            double *part = p.parts + (int64_t)(bi + blockIdx.x) * PD;
#pragma unroll
            for (int q = 0; q < MAXS; ++q) {
                const int s = b + kBxB * q;
                if (s < JS) {
#pragma unroll
                    for (int k = 0; k < NPT; ++k) {
                        const int j = F32 ? 32 * s + 4 * pg + (k >> 1) : 16 * s + 2 * pg + (k >> 1);
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int r = 2 * qperm(2 * t + e) + (k & 1);
                            if (j < J) part[j * 16 + r] = pacc[q][k][e];
                            pacc[q][k][e] = 0.0;
                        }
                    }
                }
            }
            if (b < 4) {
                double *gp = part + (int64_t)J * 16;
#pragma unroll
                for (int e = 0; e < 2; ++e) gp[(8 * mi + g) * 16 + 8 * ni + 2 * t + e] = gacc[e];
                gacc[0] = gacc[1] = 0.0;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// k_bigx_post: one CTA (256 threads) per big slice.  The P / gram / c segment
// sums are issued first (independent of w), then warp 0 solves for w, then
// F slot = P diag(w) and G slot = gram o w w^T are written.
// ---------------------------------------------------------------------------
constexpr int kPostPer = 8;  // P entries per thread: J * 16 <= 256 * kPostPer (J <= 128)
__global__ void __launch_bounds__(256) k_bigx_post(BigxParams p) {
    constexpr int RB = kBxRB, LDV = RB + 2, LDL = RB + 1;
    __shared__ double vtv_s[RB * LDV];
    __shared__ double gram_s[RB * LDL];
    __shared__ double dns[RB * LDL];
    __shared__ double lu[RB * LDL];
    __shared__ __align__(16) double vec[4 * RB + 8];  // c | w | gj scratch
    __shared__ int piv[RB];
    // Launched behind the small-row F GEMM, which triggers only after its own
    // pdl_wait: k_bigx's partials are complete.  This kernel touches nothing the
    // F GEMM does, so it runs beside it and waits only at its end.  On the fused
    // small-slice path nothing runs between k_bigx and this kernel: wait first.
    if (p.post_wait) pdl_wait();
    pdl_trigger();
    const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
    const int J = p.J, R = p.R;
    const int nsmall = __ldcg(p.plan_counts), nbig = __ldcg(p.plan_counts + 1);
    const int bi = blockIdx.x;
    if (bi >= nbig) {
        pdl_wait();
        return;
    }
    const int4 mt = __ldcg(p.meta + nsmall + bi);
    const int m = mt.w;
    const int wrow = mt.z & 0x7fffffff;
    const bool fresh = mt.z < 0;
    const int64_t T = p.T, G = p.G;
    const int64_t c0 = cta_of_tile(__ldcg(p.toff + bi), T, G);
    const int64_t c1 = cta_of_tile(__ldcg(p.toff + bi + 1) - 1, T, G);
    const int64_t PD = BigxSmem::part_doubles(J);
    const double *base = p.parts + (bi + c0) * PD;
    const int nseg = (int)(c1 - c0 + 1);
    // P (J x 16) segment sums in CTA order: thread tid owns entries tid + 256 k
    double pv[kPostPer];
#pragma unroll
    for (int k = 0; k < kPostPer; ++k) pv[k] = 0.0;
    for (int sg = 0; sg < nseg; ++sg) {
#pragma unroll
        for (int k = 0; k < kPostPer; ++k) {
            const int e = tid + 256 * k;
            if (e < J * 16) pv[k] += __ldcg(base + sg * PD + e);
        }
    }
    {
        double acc = 0.0;
        for (int sg = 0; sg < nseg; ++sg) acc += __ldcg(base + sg * PD + (int64_t)J * 16 + tid);
        gram_s[(tid / 16) * LDL + tid % 16] = acc;
    }
    if (tid < 16) {
        double acc = 0.0;
        for (int sg = 0; sg < nseg; ++sg) {
            const double *cp = base + sg * PD + (int64_t)J * 16 + 256;
#pragma unroll
            for (int a = 0; a < kBxA; ++a) acc += __ldcg(cp + 16 * a + tid);
        }
        vec[tid] = tid < R ? p.lam * (fresh ? 0.0 : __ldcg(p.C + (int64_t)wrow * R + tid)) + acc : 0.0;  // c_new
    }
    for (int i = tid; i < RB * LDV; i += blockDim.x) {
        const int a = i / LDV, b = i % LDV;
        vtv_s[i] = (a < R && b < R) ? __ldcg(p.vtv + a * R + b) : 0.0;
    }
    if (tid < RB && !fresh)
        for (int z = 0; z < R; ++z)
            dns[tid * LDL + z] = tid < R ? __ldcg(p.D + (int64_t)wrow * R * R + (int64_t)z * R + tid) : 0.0;
    __syncthreads();
    // ---- D accumulation and the S-row system by warp 0 lanes 0..15 (as k_big)
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
        double wv;
        double *gbuf = vec + 2 * RB;  // RB + 2 scratch, 16-byte aligned
        bool okB = gj_solve<RB>(a, lreal ? vec[r] : 0.0, lane < RB ? gbuf : lu, r, wv);
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
            for (int z = 0; z < RB; ++z) wv = fma(-a[z], vec[z], wv);
            if (!lreal) wv = 0.0;
            if (lreal && !isfinite(wv)) report_error(p.err, m, DASH_E_NONFINITE);
        }
        __syncwarp();
        if (lreal) {
            p.Wo[(int64_t)wrow * R + r] = wv;
            if (p.final_pass) {
                p.Co[(int64_t)wrow * R + r] = vec[r];
#pragma unroll
                for (int z = 0; z < RB; ++z)
                    if (z < R) p.D[(int64_t)wrow * R * R + (int64_t)z * R + r] = dn[z];
            }
        }
        if (lane < RB) vec[RB + lane] = lreal ? wv : 0.0;
    }
    __syncthreads();
    const double *wv = vec + RB;
    if (tid < R * R) {
        const int a = tid / R, b = tid % R;
        p.G_slots[(int64_t)bi * R * R + tid] = gram_s[a * LDL + b] * wv[a] * wv[b];
    }
    double *fs = p.F_slots + (int64_t)bi * J * R;
#pragma unroll
    for (int k = 0; k < kPostPer; ++k) {
        const int e = tid + 256 * k;  // P entry (j, r) = (e / 16, e % 16)
        const int j = e >> 4, r = e & 15;
        if (e < J * 16 && r < R) fs[j * R + r] = pv[k] * wv[r];
    }
    pdl_wait();  // completion of this grid implies the F GEMM's
}
