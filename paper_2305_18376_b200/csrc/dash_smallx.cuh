// Fused small-slice path (R bucket 16, even R, FP64, J <= 128, TMA-able X):
// the per-slice phase of the SMALL slices (<= kSmallRows rows;
// _kernels.py:62-144 + stream.py:314-322) in ONE persistent kernel, replacing
// the XV GEMM, the slice solver and the F GEMM of the three-kernel chain
// (k_xv3 -> k_slices3 -> k_fgemm3: X read twice, XV / U o w round-tripped
// through HBM, a per-row gather-bound solver).
//
// Units.  The small slices are cut, in batch order, into units of whole
// consecutive slices with <= kSxRows rows and <= kSxSlices slices (a big slice
// ends a unit).  A unit's rows are contiguous in X: one TMA load of
// ceil(span / 8) boxes of 8 rows x 16 columns per 16-column strip.
// k_sx_walk cuts each 256-position chunk with 8 sequential walkers (chunk and
// walker boundaries also end a unit: deterministic, no cross-chunk state) and
// its last block scans the per-chunk counts; k_sx_copy compacts the unit list.
// Both also carry the pass prologue (V^T V, F / G snapshots, v_used).
//
// k_smallx: persistent (one CTA per SM), warp-specialised, units split evenly
// over the CTAs in order.  Per unit u:
//
//   producer  (1 warp)   TMA: X(u) for the XV step, and X(u) again for the F
//                        step kSxLook units later (an L2 hit: a few MB were
//                        streamed in between), through one kSxNST-stage ring;
//   math      (4 warps)  warp = 8-row block.  XV = X V and Y = XV P
//                        (P = vtv^{-1}) on DMMA; then, with the slices' ridge
//                        terms d and 1/s from the solver's table, the Neumann
//                        form of the A solve (see k_slices3):
//                            U = S^{-1} (Y - (Y o d) P + ((Y o d) P o d) P)
//                        by two more small DMMA products straight from the
//                        accumulator fragments -> U tile; XV tile for c;
//                        kSxLook units later F += X^T (U o w) (DMMA, 2x2
//                        parity blocks) from the solver's US tile;
//   solver    (kSxSW warps, unit u -> warp u mod kSxSW; two slices per warp,
//              16-lane groups, lane r = rank index r):
//                        prep: s (W row; 1 for a new slice in pass 0), the
//                        ridge shift, d_r = sh / s_r^2, 1/s_r, the Neumann
//                        test per slice -> table; after the math warps' U:
//                        slices failing the test get the exact sweep (LU
//                        fallback) U rows; c = lam c_old + sum xv o u,
//                        gram = sum u u^T, D = lam D + gram, B = vtv o D +
//                        shift I solved by Gauss-Jordan (LU fallback) -> w;
//                        W / C / D rows; U rows -> U_out; U o w -> US tile;
//                        G += gram o w w^T in registers.
//
// Per-unit slots (kSxSlots): XV tile, U / US tile, table, header, with
// mbarriers prep (solver -> math), uready (math -> solver), usready (solver
// -> math) and sfree (math F done -> slot reusable).  F is one J x R slot per
// CTA, G one R x R slot per CTA (solver groups summed in fixed order):
// deterministic, no FP64 atomics.
// (included inside dash_update.cu's anonymous namespace, after dash_bigx.cuh)
#pragma once

constexpr int kSxRows = 32;          // rows per unit (max)
constexpr int kSxSlices = 16;        // slices per unit (max)
constexpr int kSxChunk = 256;        // batch positions per planner block
constexpr int kSxWalkers = 8;        // sequential walkers per planner block (32 positions each)
constexpr int kSxNST = 3;            // X ring stages
constexpr int kSxSlots = 6;          // units in flight
constexpr int kSxLook = kSxSlots - 1;  // the math warps' XV runs this many units ahead of F
constexpr int kSxMW = 4;             // math warps (one 8-row block each)
constexpr int kSxSW = kSxSlots;      // solver warps
constexpr int kSxThreads = (kSxMW + kSxSW + 1) * 32;
constexpr int kSxTP = 18;            // XV / U tile pitch (doubles): conflict-free fragment stores and row reads

struct SxSmem {
    static constexpr int JSM = 8;                        // strips (J <= 128)
    static constexpr int SD = JSM * 512;                 // doubles per ring stage (32 rows x 128 columns)
    static constexpr int VTP = JSM * 16 + 8;             // V^T pitch
    static constexpr int TILE = kSxRows * kSxTP;
    static constexpr int TBL = kSxSlices * 32;           // per slice: d[16] | sinv[16]
    static constexpr int HDR = 16;                       // int4 desc | fastmask | fast2 | rowslice[32] (bytes)
    static constexpr int SLOT = 2 * TILE + TBL + HDR;
    static constexpr int SWS = 2 * 18 + 16 * 17 + 8;     // per solver warp: 2 gather bufs | lu | piv
    static constexpr int OFF_VT = kSxNST * SD;
    static constexpr int OFF_P = OFF_VT + 16 * VTP;      // P = vtv^{-1} (16 x 16) | ||P||_inf | ok
    static constexpr int OFF_VTV = OFF_P + 264;
    static constexpr int OFF_SLOT = OFF_VTV + 16 * 18;
    static constexpr int OFF_SW = OFF_SLOT + kSxSlots * SLOT;
    static constexpr int OFF_BAR = OFF_SW + kSxSW * SWS;
    static constexpr int NBAR = 2 * kSxNST + 4 * kSxSlots;
    static constexpr size_t bytes() { return 1024 + sizeof(double) * OFF_BAR + 8 * NBAR; }
    static_assert(OFF_VT % 128 == 0, "ring stages stay 1 KB aligned");
    static_assert(SLOT % 2 == 0 && SWS % 2 == 0 && OFF_SLOT % 2 == 0 && OFF_SW % 2 == 0, "16-byte alignment");
};
static_assert(SxSmem::bytes() <= 227 * 1024, "k_smallx shared memory");

struct SxParams {
    const int4 *units;         // compacted unit list: {m0, q, a, span}
    const int *nunits;         // total units (device)
    const int64_t *row_ptr;
    const int32_t *state_row;
    const uint8_t *is_new;
    const double *V;           // J x R
    const double *vtv;         // R x R (planner prologue)
    double *W, *C, *D;         // state rows
    double *U;                 // U_out (N x R)
    double *F_slots;           // gridDim.x x J x R
    double *G_slots;           // gridDim.x x R x R
    unsigned long long *err;
    unsigned int *fallbacks;
    int J, R;
    double lam, eps;
    int pass, final_pass, sweep_only;
};

// ---------------------------------------------------------------------------
// planner: units per 256-position chunk (+ the pass prologue in extra blocks)
// ---------------------------------------------------------------------------
struct SxPlan {
    const int64_t *row_ptr;
    int M, nch;
    int4 *tmp;                 // nch x kSxChunk: units of chunk c at c * kSxChunk
    int *counts;               // nch
    int *choff;                // nch + 1: exclusive scan of counts (last block)
    int4 *units;               // compacted (k_sx_copy)
    int *nunits;
    unsigned int *done;        // last-block-done counter (reset by the last block)
};

__device__ __forceinline__ void sx_prologue(const FusedPrologue &pro, const double *V, int J, int R, int blk,
                                            int nblk) {
    // blocks [0, nvb): vtv, one warp per entry (fixed-order tree: deterministic and
    // exactly symmetric); the rest copy the snapshots / v_used
    const int nvb = (R * R + 7) / 8;
    if (blk < nvb) {
        const int p = blk * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
        if (p < R * R) {
            const int r = p / R, z = p % R;
            double a0 = 0.0, a1 = 0.0;
            for (int j = lane; j < J; j += 64) {
                a0 = fma(V[(int64_t)j * R + r], V[(int64_t)j * R + z], a0);
                if (j + 32 < J) a1 = fma(V[(int64_t)(j + 32) * R + r], V[(int64_t)(j + 32) * R + z], a1);
            }
            double acc = a0 + a1;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(FULL_MASK, acc, off);
            if (lane == 0) pro.vtv[p] = acc;
        }
        return;
    }
    const int tid = (blk - nvb) * blockDim.x + threadIdx.x, nt = (nblk - nvb) * blockDim.x;
    if (pro.snap) {
        for (int i = tid; i < J * R; i += nt) pro.F_snap[i] = pro.F[i];
        for (int i = tid; i < R * R; i += nt) pro.G_snap[i] = pro.G[i];
    }
    if (pro.last)
        for (int i = tid; i < J * R; i += nt) pro.v_used[i] = V[i];
}

__host__ __device__ inline int sx_prologue_blocks(int R) { return (R * R + 7) / 8 + 4; }

__global__ void __launch_bounds__(256) k_sx_walk(SxPlan pl, FusedPrologue pro, const double *V, int J, int R) {
    pdl_trigger();
    const int tid = threadIdx.x;
    if ((int)blockIdx.x >= pl.nch) {  // prologue blocks: inputs final since the update's first kernel started
        sx_prologue(pro, V, J, R, blockIdx.x - pl.nch, gridDim.x - pl.nch);
        pdl_wait();
        return;
    }
    __shared__ int64_t rp[kSxChunk + 1];
    __shared__ int4 ub[kSxChunk];
    __shared__ int uc[kSxWalkers];
    __shared__ bool last;
    const int c0 = blockIdx.x * kSxChunk;
    const int cnt = min(kSxChunk, pl.M - c0);
    for (int i = tid; i <= cnt; i += blockDim.x) rp[i] = pl.row_ptr[c0 + i];
    __syncthreads();
    constexpr int PER = kSxChunk / kSxWalkers;
    if (tid < kSxWalkers) {
        int k = 0, m0 = 0, q = 0, rows = 0;
        int64_t a = 0;
        bool open = false;
        const int p1 = min(cnt, (tid + 1) * PER);
        for (int p = tid * PER; p < p1; ++p) {
            const int64_t n = rp[p + 1] - rp[p];
            if (n > kSmallRows) {  // a big slice ends the unit
                if (open) ub[tid * PER + k++] = make_int4(m0, q, (int)a, rows);
                open = false;
                continue;
            }
            if (open && (rows + n > kSxRows || q == kSxSlices)) {
                ub[tid * PER + k++] = make_int4(m0, q, (int)a, rows);
                open = false;
            }
            if (!open) {
                open = true;
                m0 = c0 + p;
                q = 0;
                a = rp[p];
                rows = 0;
            }
            rows += (int)n;
            ++q;
        }
        if (open) ub[tid * PER + k++] = make_int4(m0, q, (int)a, rows);
        uc[tid] = k;
    }
    __syncthreads();
    {
        int off = 0, tot = 0;
        const int wk = tid / PER, kk = tid % PER;
#pragma unroll
        for (int i = 0; i < kSxWalkers; ++i) {
            if (i < wk) off += uc[i];
            tot += uc[i];
        }
        if (kk < uc[wk]) pl.tmp[(int64_t)c0 + off + kk] = ub[tid];
        if (tid == 0) pl.counts[blockIdx.x] = tot;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) last = atomicAdd(pl.done, 1u) == (unsigned)pl.nch - 1;
    __syncthreads();
    if (last) {  // exclusive scan of the chunk counts (fixed order) -> choff, nunits
        __threadfence();
        __shared__ int wsum[8];
        const int lane = tid & 31, wq = tid >> 5;
        int carry = 0;
        for (int b0 = 0; b0 < pl.nch; b0 += 256) {
            const int c = b0 + tid;
            const int v = c < pl.nch ? __ldcg(pl.counts + c) : 0;
            int inc = v;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int u = __shfl_up_sync(FULL_MASK, inc, d);
                if (lane >= d) inc += u;
            }
            if (lane == 31) wsum[wq] = inc;
            __syncthreads();
            int wb = 0, all = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (i < wq) wb += wsum[i];
                all += wsum[i];
            }
            if (c < pl.nch) pl.choff[c] = carry + wb + inc - v;
            carry += all;
            __syncthreads();
        }
        if (tid == 0) {
            pl.choff[pl.nch] = carry;
            *pl.nunits = carry;
            *pl.done = 0u;
        }
    }
    pdl_wait();
}

// one block per chunk: its units -> units[choff[c] ...]
__global__ void __launch_bounds__(256) k_sx_copy(SxPlan pl) {
    pdl_wait();
    pdl_trigger();
    const int c = blockIdx.x;
    const int n = __ldcg(pl.counts + c), o = __ldcg(pl.choff + c);
    for (int k = threadIdx.x; k < n; k += blockDim.x) pl.units[o + k] = __ldcg(pl.tmp + (int64_t)c * kSxChunk + k);
}

// ---------------------------------------------------------------------------
// k_smallx
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kSxThreads, 1) k_smallx(const __grid_constant__ CUtensorMap tmX, SxParams p) {
    using S = SxSmem;
    constexpr int RB = 16, LDV = 18;
    extern __shared__ __align__(16) double sm_raw[];
    double *sm = align1k(sm_raw);
    double *xs = sm;
    double *vt = sm + S::OFF_VT;
    double *P_s = sm + S::OFF_P;
    double *vtv_s = sm + S::OFF_VTV;
    double *slots = sm + S::OFF_SLOT;
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + S::OFF_BAR);
    uint64_t *full = bar, *empty = bar + kSxNST;
    uint64_t *prep = empty + kSxNST, *uready = prep + kSxSlots, *usready = uready + kSxSlots,
             *sfree = usready + kSxSlots;
    const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
    const int J = p.J, R = p.R;
    const int JS = (J + 15) / 16;

    pdl_wait();     // units, vtv (planner), previous pass / update complete
    pdl_trigger();  // k_bigx_pre may fill SMs as this kernel's CTAs retire

    if (tid == 0) {
        prefetch_map(&tmX);
        for (int s = 0; s < kSxNST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kSxMW);
        }
        for (int s = 0; s < kSxSlots; ++s) {
            mbar_init(&prep[s], 1);
            mbar_init(&uready[s], kSxMW);
            mbar_init(&usready[s], 1);
            mbar_init(&sfree[s], kSxMW);
        }
        fence_mbar_init();
    }
    // ring zeroed once: rows past a unit's boxes are stale but always finite
    for (int i = tid; i < kSxNST * S::SD; i += blockDim.x) xs[i] = 0.0;
    for (int i = tid; i < 16 * S::VTP; i += blockDim.x) {
        const int nn = i / S::VTP, k = i % S::VTP;
        vt[i] = (nn < R && k < J) ? __ldg(p.V + k * R + nn) : 0.0;
    }
    for (int i = tid; i < RB * LDV; i += blockDim.x) {
        const int a = i / LDV, b = i % LDV;
        vtv_s[i] = (a < R && b < R) ? __ldcg(p.vtv + a * R + b) : 0.0;
    }
    __syncthreads();
    // P = vtv^{-1} once per CTA (warp 0, both groups; group 0 writes), as k_slices3
    if (w == 0) {
        const int r = lane & 15;
        double *buf = sm + S::OFF_SW + (lane >> 4) * 18;
        const double *vrow = vtv_s + r * LDV;
        double a[RB];
        double mx = r < R ? vrow[r] : 0.0;
#pragma unroll
        for (int off = 8; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL_MASK, mx, off));
        const double im = (mx > 0.0 && isfinite(mx)) ? 1.0 / mx : 1.0;
#pragma unroll
        for (int z = 0; z < RB; ++z) a[z] = (r < R) ? ((z < R) ? vrow[z] * im : 0.0) : ((z == r) ? 1.0 : 0.0);
        const bool ok = sweep_inverse_unit<RB>(a, buf, r);
        double rs = 0.0;
#pragma unroll
        for (int z = 0; z < RB; ++z) {
            a[z] = (r < R && z < R) ? -a[z] * im : 0.0;
            rs += fabs(a[z]);
        }
#pragma unroll
        for (int off = 8; off > 0; off >>= 1) rs = fmax(rs, __shfl_xor_sync(FULL_MASK, rs, off));
        if (lane < 16) {
#pragma unroll
            for (int z = 0; z < RB; ++z) P_s[z * RB + r] = a[z];
            if (r == 0) {
                P_s[256] = rs;
                P_s[257] = (ok && isfinite(rs) && !p.sweep_only) ? 1.0 : 0.0;
            }
        }
    }
    __syncthreads();

    const int U = __ldcg(p.nunits);
    const int G = gridDim.x;
    const int u0 = (int)((int64_t)U * blockIdx.x / G), u1 = (int)((int64_t)U * (blockIdx.x + 1) / G);
    const int nmine = u1 - u0;
    const int4 *units = p.units + u0;
    const int nitems = nmine > 0 ? 2 * nmine : 0;  // XV(u) and F(u) per unit, in the math warps' order
    // item i of the sequence: for v = 0 .. nmine + kSxLook - 1: XV(v) if v < nmine, then F(v - kSxLook) if v >= kSxLook

    if (w == kSxMW + kSxSW) {  // ---------------- producer
        if (lane == 0 && nmine > 0) {
            int64_t item = 0;
            auto load = [&](int u) {
                const int4 d = __ldcg(units + u);
                const int st = (int)(item % kSxNST);
                if (item >= kSxNST) mbar_wait(&empty[st], (uint32_t)(((item / kSxNST) - 1) & 1));
                const int nb = (d.w + 7) >> 3;
                mbar_arrive_expect_tx(&full[st], (uint32_t)(JS * nb) * 1024u);
                for (int s = 0; s < JS; ++s)
                    for (int b = 0; b < nb; ++b)
                        tma_load_2d(xs + st * S::SD + s * 512 + b * 128, &tmX, 16 * s, d.z + 8 * b, &full[st]);
                ++item;
            };
            for (int v = 0; v < nmine + kSxLook; ++v) {
                if (v < nmine) load(v);
                if (v >= kSxLook) load(v - kSxLook);
            }
        }
        return;
    }
    const int g = lane >> 2, t = lane & 3;
    if (w < kSxMW) {  // ---------------- math warps
        const int mb = w;
        const int pg = qperm(g);
        const int xrow = 8 * mb + pg;  // this lane's row of the unit (A-fragment / C-fragment row)
        double pf[4][2];               // B fragments of P in the permuted K order (P symmetric)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
#pragma unroll
            for (int nb = 0; nb < 2; ++nb) pf[kk][nb] = P_s[(8 * nb + g) * 16 + 8 * (kk >> 1) + 2 * t + (kk & 1)];
        double facc[2][4][2];
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
            for (int k = 0; k < 4; ++k) facc[q][k][0] = facc[q][k][1] = 0.0;
        int64_t item = 0;
        for (int v = 0; v < nmine + kSxLook; ++v) {
            if (v < nmine) {  // ---- XV(v), Y, U
                const int u = v, slot = u % kSxSlots, use = u / kSxSlots;
                const int st = (int)(item % kSxNST);
                mbar_wait(&full[st], (uint32_t)((item / kSxNST) & 1));
                ++item;
                const double *xt = xs + st * S::SD;
                double xa[2][4][2];
#pragma unroll
                for (int nb = 0; nb < 2; ++nb)
#pragma unroll
                    for (int c = 0; c < 4; ++c) xa[nb][c][0] = xa[nb][c][1] = 0.0;
#pragma unroll
                for (int s = 0; s < S::JSM; ++s) {
                    if (s < JS) {
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const double2 a = *reinterpret_cast<const double2 *>(xt + s * 512 + swz(xrow, 4 * h + t));
#pragma unroll
                            for (int nb = 0; nb < 2; ++nb) {
                                const double2 b = *reinterpret_cast<const double2 *>(vt + (8 * nb + g) * S::VTP +
                                                                                     16 * s + 8 * h + 2 * t);
                                dmma884(xa[nb][2 * h], a.x, b.x);
                                dmma884(xa[nb][2 * h + 1], a.y, b.y);
                            }
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[st]);
                double xv[2][2];
#pragma unroll
                for (int nb = 0; nb < 2; ++nb)
#pragma unroll
                    for (int e = 0; e < 2; ++e) xv[nb][e] = (xa[nb][0][e] + xa[nb][1][e]) + (xa[nb][2][e] + xa[nb][3][e]);
                // Y = XV P: A fragment of K step kk = this lane's XV value xv[kk >> 1][kk & 1]
                double ya[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
#pragma unroll
                    for (int nb = 0; nb < 2; ++nb) dmma884(ya[nb], xv[kk >> 1][kk & 1], pf[kk][nb]);
                double *sl = slots + slot * S::SLOT;
                double *xvt = sl, *ut = sl + S::TILE, *tbl = sl + 2 * S::TILE;
                const int *hdr = reinterpret_cast<const int *>(tbl + S::TBL);
                if (use >= 1) mbar_wait(&sfree[slot], (uint32_t)((use - 1) & 1));  // F(u - kSxSlots) done
#pragma unroll
                for (int nb = 0; nb < 2; ++nb)
                    *reinterpret_cast<double2 *>(xvt + xrow * kSxTP + 8 * nb + 2 * t) = make_double2(xv[nb][0], xv[nb][1]);
                mbar_wait(&prep[slot], (uint32_t)(use & 1));
                const int span = hdr[3];
                const int fast2 = hdr[5];
                const bool valid = xrow < span;
                const int k = valid ? (int)reinterpret_cast<const uint8_t *>(hdr + 8)[xrow] : 0;
                const double *dk = tbl + k * 32;
                double dd[2][2], si[2][2];
#pragma unroll
                for (int nb = 0; nb < 2; ++nb) {
                    const double2 a = *reinterpret_cast<const double2 *>(dk + 8 * nb + 2 * t);
                    const double2 b = *reinterpret_cast<const double2 *>(dk + 16 + 8 * nb + 2 * t);
                    dd[nb][0] = valid ? a.x : 0.0;
                    dd[nb][1] = valid ? a.y : 0.0;
                    si[nb][0] = b.x;
                    si[nb][1] = b.y;
                }
                double c1[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
#pragma unroll
                    for (int nb = 0; nb < 2; ++nb)
                        dmma884(c1[nb], ya[kk >> 1][kk & 1] * dd[kk >> 1][kk & 1], pf[kk][nb]);  // (Y o d) P
                double c2[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
                if (fast2) {  // unit-uniform
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
#pragma unroll
                        for (int nb = 0; nb < 2; ++nb)
                            dmma884(c2[nb], c1[kk >> 1][kk & 1] * dd[kk >> 1][kk & 1], pf[kk][nb]);
                }
#pragma unroll
                for (int nb = 0; nb < 2; ++nb) {
                    double u2[2];
#pragma unroll
                    for (int e = 0; e < 2; ++e) u2[e] = valid ? ((ya[nb][e] - c1[nb][e]) + c2[nb][e]) * si[nb][e] : 0.0;
                    *reinterpret_cast<double2 *>(ut + xrow * kSxTP + 8 * nb + 2 * t) = make_double2(u2[0], u2[1]);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&uready[slot]);
            }
            if (v >= kSxLook) {  // ---- F(v - kSxLook) += X^T US
                const int u = v - kSxLook, slot = u % kSxSlots, use = u / kSxSlots;
                const int st = (int)(item % kSxNST);
                mbar_wait(&full[st], (uint32_t)((item / kSxNST) & 1));
                ++item;
                mbar_wait(&usready[slot], (uint32_t)(use & 1));
                const double *xt = xs + st * S::SD;
                const double *ub = slots + slot * S::SLOT + S::TILE;
#pragma unroll
                for (int kk = 0; kk < kSxRows / 4; ++kk) {
                    const int row = 4 * kk + t;
                    const double2 bu = *reinterpret_cast<const double2 *>(ub + row * kSxTP + 2 * pg);
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const int s = mb + 4 * q;
                        if (s < JS) {
                            const double2 a = *reinterpret_cast<const double2 *>(xt + s * 512 + swz(row, pg));
                            dmma884(facc[q][0], a.x, bu.x);
                            dmma884(facc[q][1], a.x, bu.y);
                            dmma884(facc[q][2], a.y, bu.x);
                            dmma884(facc[q][3], a.y, bu.y);
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&empty[st]);
                    mbar_arrive(&sfree[slot]);
                }
            }
        }
        // F slot of this CTA (every entry written by exactly one lane; zeros if no units)
        double *fs = p.F_slots + (int64_t)blockIdx.x * J * R;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int s = mb + 4 * q;
            if (s < JS) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int j = 16 * s + 2 * pg + (k >> 1);
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int r = 2 * qperm(2 * t + e) + (k & 1);
                        if (j < J && r < R) fs[(int64_t)j * R + r] = facc[q][k][e];
                    }
                }
            }
        }
        (void)nitems;
        asm volatile("bar.sync 1, %0;" ::"n"((kSxMW + kSxSW) * 32) : "memory");
        return;
    }
    // ---------------- solver warps
    const int ws = w - kSxMW;
    const int r = lane & 15, gl = lane >> 4;
    double *wsm = sm + S::OFF_SW + ws * S::SWS;
    double *buf = wsm + gl * 18;
    double *lu = wsm + 36;
    int *piv = reinterpret_cast<int *>(lu + 16 * 17);
    const double *vrow = vtv_s + r * LDV;
    const double pnorm = P_s[256];
    const bool pok = P_s[257] != 0.0;
    double gacc[RB];
#pragma unroll
    for (int z = 0; z < RB; ++z) gacc[z] = 0.0;
    for (int u = ws; u < nmine; u += kSxSW) {
        const int slot = u % kSxSlots, use = u / kSxSlots;
        const int4 d = __ldcg(units + u);
        const int m0 = d.x, q = d.y, a0 = d.z, span = d.w;
        double *sl = slots + slot * S::SLOT;
        double *xvt = sl, *ut = sl + S::TILE, *tbl = sl + 2 * S::TILE;
        int *hdr = reinterpret_cast<int *>(tbl + S::TBL);
        uint8_t *rowslice = reinterpret_cast<uint8_t *>(hdr + 8);
        if (use >= 1) mbar_wait(&sfree[slot], (uint32_t)((use - 1) & 1));
        // ---- prep: s, ridge shift, d = sh / s^2, 1/s, Neumann test (k_slices3's) -> table
        unsigned fastmask = 0u;
        bool any2 = false;
        for (int pr = 0; pr < q; pr += 2) {
            const int j = pr + gl;
            const bool act = j < q;
            const int m = m0 + (act ? j : 0);
            const int wrow = __ldg(p.state_row + m);
            const bool fresh = __ldg(p.is_new + m) != 0;
            const bool real = act && r < R;
            const double s_r = real ? ((fresh && p.pass == 0) ? 1.0 : __ldcg(p.W + (int64_t)wrow * R + r)) : 0.0;
            double s_all[RB];
            group_gather<RB>(s_r, buf, r, s_all);
            double q4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int z = 0; z < RB; ++z)
                if (z < R) q4[z & 3] = fma(vtv_s[z * LDV + z] * s_all[z], s_all[z], q4[z & 3]);
            const double sh = p.eps * ((q4[0] + q4[1]) + (q4[2] + q4[3])) / R;
            double qv = 0.0, isr = 0.0;
            bool bad = false;
            if (real) {
                isr = rcp_nr(s_r);
                qv = isr * isr;
                bad = !(s_r != 0.0) || !isfinite(qv);
            }
            double qm = bad ? INFINITY : qv;
#pragma unroll
            for (int off = 8; off > 0; off >>= 1) qm = fmax(qm, __shfl_xor_sync(FULL_MASK, qm, off));
            const double rho = sh * qm * pnorm;
            const bool fast = act && pok && rho <= kS3Neumann;  // NaN / inf -> exact path
            const unsigned fb = __ballot_sync(FULL_MASK, fast && r == 0);
            fastmask |= ((fb & 1u) ? 1u : 0u) << pr;
            fastmask |= ((fb >> 16) & 1u) << (pr + 1);
            any2 = any2 || __any_sync(FULL_MASK, fast && !(rho <= kS3Neumann1));
            if (act) {
                tbl[j * 32 + r] = real ? sh * qv : 0.0;
                tbl[j * 32 + 16 + r] = real ? isr : 0.0;
                const int64_t rb = __ldg(p.row_ptr + m) - a0, n = __ldg(p.row_ptr + m + 1) - __ldg(p.row_ptr + m);
                for (int64_t i = r; i < n; i += 16) rowslice[rb + i] = (uint8_t)j;
            }
        }
        if (lane == 0) {
            hdr[0] = m0;
            hdr[1] = q;
            hdr[2] = a0;
            hdr[3] = span;
            hdr[4] = (int)fastmask;
            hdr[5] = any2 ? 1 : 0;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&prep[slot]);
        mbar_wait(&uready[slot], (uint32_t)(use & 1));
        // ---- per slice pair
        for (int pr = 0; pr < q; pr += 2) {
            const int j = pr + gl;
            const bool act = j < q;
            const int m = m0 + (act ? j : 0);
            const int wrow = __ldg(p.state_row + m);
            const bool fresh = __ldg(p.is_new + m) != 0;
            const bool real = act && r < R;
            const int64_t rg = __ldg(p.row_ptr + m);
            const int rb = (int)(rg - a0);
            const int n = act ? (int)(__ldg(p.row_ptr + m + 1) - rg) : 0;
            // state loads first (latency overlaps the rows loop)
            const double cold = (real && !fresh) ? __ldcg(p.C + (int64_t)wrow * R + r) : 0.0;
            double dold[RB];
#pragma unroll
            for (int z = 0; z < RB; ++z)
                dold[z] = (real && !fresh && z < R) ? __ldcg(p.D + (int64_t)wrow * R * R + (int64_t)z * R + r) : 0.0;
            const double s_r = real ? ((fresh && p.pass == 0) ? 1.0 : __ldcg(p.W + (int64_t)wrow * R + r)) : 0.0;
            const bool fast = act && ((fastmask >> j) & 1u);
            int nmax = n;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) nmax = max(nmax, __shfl_xor_sync(FULL_MASK, nmax, off));
            // ---- slices failing the Neumann test: exact A solve (sweep, LU fallback), U rows rewritten
            if (__any_sync(FULL_MASK, act && !fast)) {
                const bool ex = act && !fast;
                double s_all[RB];
                group_gather<RB>(s_r, buf, r, s_all);
                double sh;
                {
                    double q4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                    for (int z = 0; z < RB; ++z)
                        if (z < R) q4[z & 3] = fma(vtv_s[z * LDV + z] * s_all[z], s_all[z], q4[z & 3]);
                    sh = p.eps * ((q4[0] + q4[1]) + (q4[2] + q4[3])) / R;
                }
                const double dg = real ? sh : 1.0;
                double mx = vrow[r] * s_r * s_r + dg;
#pragma unroll
                for (int off = 8; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL_MASK, mx, off));
                double im = (mx > 0.0 && isfinite(mx)) ? 1.0 / mx : 1.0;
                double a[RB];
                {
                    const double sr_im = s_r * im, dg_im = dg * im;
#pragma unroll
                    for (int z = 0; z < RB; ++z) a[z] = vrow[z] * sr_im * s_all[z] + ((z == r) ? dg_im : 0.0);
                }
                const bool okA = sweep_inverse_unit<RB>(a, buf, r);
                if (!okA) im = 1.0;
                if (__any_sync(FULL_MASK, ex && !okA)) {
                    const bool need = ex && !okA;
#pragma unroll
                    for (int z = 0; z < RB; ++z)
                        if (need) a[z] = vrow[z] * s_r * s_all[z] + ((z == r) ? dg : 0.0);
                    if (need && r == 0) atomicAdd(p.fallbacks, 1u);
                    const bool okLU = lu_fallback_seq<RB>(a, lu, piv, r, R, need);
                    if (need && r == 0 && !okLU) report_error(p.err, m, DASH_E_SINGULAR);
                }
#pragma unroll
                for (int z = 0; z < RB; ++z) a[z] *= s_all[z];
                for (int i = 0; i < nmax; ++i) {
                    double u = 0.0;
                    if (ex && i < n) {
                        const double *xr = xvt + (rb + i) * kSxTP;
                        double xrow_v[RB];
#pragma unroll
                        for (int z = 0; z < RB / 2; ++z) {
                            const double2 t2 = *reinterpret_cast<const double2 *>(xr + 2 * z);
                            xrow_v[2 * z] = t2.x;
                            xrow_v[2 * z + 1] = t2.y;
                        }
                        u = neg_dot4<RB>(a, xrow_v, R) * im;
                        if (!(r < R)) u = 0.0;
                    }
                    __syncwarp();
                    if (ex && i < n) ut[(rb + i) * kSxTP + r] = u;
                }
                __syncwarp();
            }
            // ---- rows: U -> U_out, c, gram (_kernels.py:98-115)
            double c = 0.0, gram[RB];
#pragma unroll
            for (int z = 0; z < RB; ++z) gram[z] = 0.0;
            for (int i = 0; i < nmax; ++i) {
                if (i < n) {
                    const double *urw = ut + (rb + i) * kSxTP;
                    double ua[RB];
#pragma unroll
                    for (int z = 0; z < RB / 2; ++z) {
                        const double2 t2 = *reinterpret_cast<const double2 *>(urw + 2 * z);
                        ua[2 * z] = t2.x;
                        ua[2 * z + 1] = t2.y;
                    }
                    const double ur = ua[r];
#pragma unroll
                    for (int z = 0; z < RB; ++z) gram[z] = fma(ur, ua[z], gram[z]);
                    if (real) {
                        c = fma(xvt[(rb + i) * kSxTP + r], ur, c);
                        p.U[(rg + i) * R + r] = ur;
                    }
                }
            }
            // ---- c, D accumulation and the S-row system (_kernels.py:103-135)
            const double cn = real ? p.lam * cold + c : 0.0;
            double dn[RB];
            double drr = 0.0;
#pragma unroll
            for (int z = 0; z < RB; ++z) {
                dn[z] = (real && z < R) ? p.lam * dold[z] + gram[z] : 0.0;
                if (z == r) drr = dn[z];
            }
            double sh2;
            {
                double vdd[RB];
                group_gather<RB>(real ? vrow[r] * drr : 0.0, buf, r, vdd);
                double dsum = 0.0;
#pragma unroll
                for (int z = 0; z < RB; ++z)
                    if (z < R) dsum += vdd[z];
                sh2 = p.eps * dsum / R;
            }
            double a[RB];
            {
                const double dg2 = real ? sh2 : 1.0;
#pragma unroll
                for (int z = 0; z < RB; ++z) a[z] = vrow[z] * dn[z] + ((z == r) ? dg2 : 0.0);
            }
            double wv;
            const bool okB = gj_solve<RB>(a, cn, buf, r, wv);
            if (!real) wv = 0.0;
            bool gok = okB && isfinite(wv);
            {
                const unsigned bal = __ballot_sync(FULL_MASK, !gok);
                const unsigned gmask = 0xffffu << (gl * 16);
                gok = (bal & gmask) == 0;
            }
            if (__any_sync(FULL_MASK, !gok && act)) {
                const bool need = !gok && act;
                const double dg2 = real ? sh2 : 1.0;
#pragma unroll
                for (int z = 0; z < RB; ++z)
                    if (need) a[z] = vrow[z] * dn[z] + ((z == r) ? dg2 : 0.0);
                if (need && r == 0) atomicAdd(p.fallbacks, 1u);
                const bool okLU = lu_fallback_seq<RB>(a, lu, piv, r, R, need);
                if (need && r == 0 && !okLU) report_error(p.err, m, DASH_E_SINGULAR);
                double call[RB];
                group_gather<RB>(cn, buf, r, call);
                double wv2 = 0.0;
#pragma unroll
                for (int z = 0; z < RB; ++z) wv2 = fma(-a[z], call[z], wv2);
                if (need) wv = real ? wv2 : 0.0;
                if (need && real && !isfinite(wv)) report_error(p.err, m, DASH_E_NONFINITE);
            }
            if (real) {
                p.W[(int64_t)wrow * R + r] = wv;
                if (p.final_pass) {
                    p.C[(int64_t)wrow * R + r] = cn;
#pragma unroll
                    for (int z = 0; z < RB; ++z)
                        if (z < R) p.D[(int64_t)wrow * R * R + (int64_t)z * R + r] = dn[z];
                }
            }
            __syncwarp();  // every lane's gram row reads are done before US overwrites U
            for (int i = 0; i < n; ++i) ut[(rb + i) * kSxTP + r] *= wv;  // padded lanes: wv = 0
            double wa[RB];
            group_gather<RB>(wv, buf, r, wa);
            if (act) {
#pragma unroll
                for (int z = 0; z < RB; ++z) gacc[z] = fma(gram[z] * wv, wa[z], gacc[z]);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&usready[slot]);
    }
    // ---- per-CTA G slot: solver groups summed in fixed order (slot tiles reused as scratch)
    asm volatile("bar.sync 1, %0;" ::"n"((kSxMW + kSxSW) * 32) : "memory");
    double *red = slots;  // kSxSW x 2 groups x 16 x 16 <= kSxSlots x SLOT
#pragma unroll
    for (int z = 0; z < RB; ++z) red[((ws * 2 + gl) * 16 + r) * 16 + z] = gacc[z];
    asm volatile("bar.sync 2, %0;" ::"n"(kSxSW * 32) : "memory");
    double *gs = p.G_slots + (int64_t)blockIdx.x * R * R;
    for (int i = tid - kSxMW * 32; i < R * R; i += kSxSW * 32) {
        const int a = i / R, b = i % R;
        double acc = 0.0;
        for (int k = 0; k < 2 * kSxSW; ++k) acc += red[(k * 16 + a) * 16 + b];
        gs[i] = acc;
    }
}

int launch_smallx(dash_ctx *ctx, cudaStream_t st, const CUtensorMap &map8, const SxParams &sp, int grid) {
    const size_t smem = SxSmem::bytes();
    ensure_smem_attr(k_smallx, smem);
    return launch_k(true, k_smallx, grid, kSxThreads, smem, st, map8, sp);
}
