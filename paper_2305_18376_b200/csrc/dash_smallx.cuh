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
constexpr int kSxNST = 2;            // X ring stages
constexpr int kSxSlots = 6;          // units in flight (XV / U tiles)
constexpr int kSxLook = kSxSlots - 1;  // the math warps' XV runs this many units ahead of F
constexpr int kSxMW = 4;             // math warps (one 8-row block each)
constexpr int kSxSW = 10;            // solver warps (slice pairs round-robin over the unit sequence)
constexpr int kSxThreads = (kSxMW + kSxSW + 2) * 32;  // + TMA warp + metadata warp: 16 warps, 128 registers
constexpr int kSxTP = 18;            // XV / U tile pitch (doubles): conflict-free fragment stores and row reads

constexpr int kSxNM = 8;              // per-unit metadata slots (staged by the metadata warp ahead of the math)
// unit record (planner -> producer; also the layout of a metadata slot's header), ints:
// [0..3] {m0, q, a, span} | [4..20] rp[q+1] (unit-local first rows) | [21..36] state rows |
// [37..40] is_new bytes | [41] "second Neumann term" flag (producer) | pad
constexpr int kSxRec = 48;

struct SxSmem {
    static constexpr int JSM = 8;                        // strips (J <= 128)
    static constexpr int SD = JSM * 512;                 // doubles per ring stage (32 rows x 128 columns)
    static constexpr int VTP = JSM * 16 + 8;             // V^T pitch
    static constexpr int TILE = kSxRows * kSxTP;
    static constexpr int SLOT = 2 * TILE;                // XV tile | U / US tile
    // per-unit metadata (producer -> math, solver): int desc[4] | rp[kSxSlices + 1] (unit-local first
    // rows) | wrow[kSxSlices] | fresh[kSxSlices] (bytes) -> 24 doubles, then the slices' W rows (16 each)
    static constexpr int MHDR = 24;
    static constexpr int MSH = MHDR + kSxSlices * 16;    // per slice: ridge shift sh
    static constexpr int META = MSH + kSxSlices;
    static constexpr int LUS = 16 * 17 + 8 + 4;          // shared LU fallback scratch | piv | lock
    static constexpr int SWS = 2 * 18 + 2 * 256;         // per solver warp: 2 gather bufs | 2 D stages
    static constexpr int OFF_VT = kSxNST * SD;
    static constexpr int OFF_P = OFF_VT + 16 * VTP;      // P = vtv^{-1} (16 x 16) | ||P||_inf | ok
    static constexpr int OFF_VTV = OFF_P + 264;
    static constexpr int OFF_SLOT = OFF_VTV + 16 * 18;
    static constexpr int OFF_META = OFF_SLOT + kSxSlots * SLOT;
    static constexpr int OFF_LU = OFF_META + kSxNM * META;
    static constexpr int OFF_SW = OFF_LU + LUS;
    static constexpr int OFF_BAR = OFF_SW + kSxSW * SWS;
    static constexpr int NBAR = 2 * kSxNST + 2 * kSxSlots + 2 * kSxNM;
    static constexpr size_t bytes() { return 1024 + sizeof(double) * OFF_BAR + 8 * NBAR; }
    static_assert(OFF_VT % 128 == 0, "ring stages stay 1 KB aligned");
    static_assert(SLOT % 2 == 0 && META % 2 == 0 && LUS % 2 == 0 && SWS % 2 == 0 && OFF_SLOT % 2 == 0 &&
                      OFF_META % 2 == 0 && OFF_SW % 2 == 0, "16-byte alignment");
};
static_assert(SxSmem::bytes() <= 227 * 1024, "k_smallx shared memory");

#ifdef DASH_SX_TRACE
__device__ long long g_sxtrace[148 * 64 * 8];  // [cta][unit < 64][event]
#define SX_T(u, e)                                                                                \
    do {                                                                                          \
        if ((u) < 64 && blockIdx.x < 148) g_sxtrace[(blockIdx.x * 64 + (u)) * 8 + (e)] = clock64(); \
    } while (0)
__device__ long long g_sxtrace2[64 * 8 * 8];
#define SX_P(e)                                                                                 \
    do {                                                                                        \
        if (blockIdx.x == 0 && ws == 0 && lane == 0 && n_pairs <= 16) g_sxtrace2[1024 + (n_pairs - 1) * 16 + (e)] = clock64(); \
    } while (0)
#define SX_M(u, e)                                                                    \
    do {                                                                              \
        if (blockIdx.x == 0 && mb == 0 && lane == 0 && (u) < 64) g_sxtrace2[(u) * 8 + (e)] = clock64(); \
    } while (0)
#else
#define SX_P(e) \
    do {        \
    } while (0)
#define SX_M(u, e) \
    do {           \
    } while (0)
#define SX_T(u, e) \
    do {           \
    } while (0)
#endif

struct SxParams {
    const int *units;          // unit records (kSxRec ints each, see k_sx_copy)
    const int *nunits;         // total units (device)
    const int64_t *row_ptr;
    const int32_t *state_row;
    const uint8_t *is_new;
    const double *V;           // J x R
    const double *vtv;         // R x R (planner prologue)
    double *W, *C, *D;         // state rows
    double *U;                 // U_out (N x R)
    double *US;                // U o w (N x R): operand of the F GEMM (k_fgemm3, which also forms G)
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
    int *units;                // compacted unit records (k_sx_copy), kSxRec ints each
    int *nunits;
    unsigned int *done;        // last-block-done counter (reset by the last block)
    const int32_t *state_row;
    const uint8_t *is_new;
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

// one block per chunk, one thread per unit: the chunk's units -> records
// units[(choff[c] + k) * kSxRec]: desc, unit-local row offsets, state rows, flags
__global__ void __launch_bounds__(256) k_sx_copy(SxPlan pl) {
    pdl_wait();
    pdl_trigger();
    const int c = blockIdx.x;
    const int n = __ldcg(pl.counts + c), o = __ldcg(pl.choff + c);
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        const int4 d = __ldcg(pl.tmp + (int64_t)c * kSxChunk + k);
        int *rec = pl.units + (int64_t)(o + k) * kSxRec;
        int v[kSxRec];
#pragma unroll
        for (int i = 0; i < kSxRec; ++i) v[i] = 0;
        v[0] = d.x;
        v[1] = d.y;
        v[2] = d.z;
        v[3] = d.w;
#pragma unroll
        for (int j = 0; j <= kSxSlices; ++j)
            if (j <= d.y) v[4 + j] = (int)(pl.row_ptr[d.x + j] - d.z);
        unsigned fb[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int j = 0; j < kSxSlices; ++j)
            if (j < d.y) {
                v[4 + kSxSlices + 1 + j] = pl.state_row[d.x + j];
                fb[j >> 2] |= (pl.is_new[d.x + j] ? 1u : 0u) << (8 * (j & 3));
            }
#pragma unroll
        for (int i = 0; i < 4; ++i) v[4 + 2 * kSxSlices + 1 + i] = (int)fb[i];
#pragma unroll
        for (int i = 0; i < kSxRec / 4; ++i)
            reinterpret_cast<int4 *>(rec)[i] = make_int4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    }
}

// P = vtv^{-1} (row-distributed sweep on the scaled Gram, as k_slices3), its
// infinity norm and an ok flag -> P_s[0..255] | P_s[256] | P_s[257].  Warp-wide.
__device__ __noinline__ void sx_inverse_vtv(const double *vtv_s, double *P_s, double *buf, int R, int sweep_only) {
    constexpr int RB = 16, LDV = 18;
    const int lane = lane_id(), r = lane & 15;
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
            P_s[257] = (ok && isfinite(rs) && !sweep_only) ? 1.0 : 0.0;
        }
    }
    __syncwarp();
}

// Cold path of the solver pair loop: the slices with `ex` set failed the
// Neumann test; their U rows are recomputed from the XV tile by the exact
// A = vtv o s s^T + shift I solve (scaled sweep, LU fallback; k_slices3's
// chain) and written over the math warps' tile rows.  Warp-wide (both groups).
__device__ __noinline__ void sx_exact_rows(const double *vtv_s, double *buf, double *lu, int *piv,
                                           const double *xvt, double *ut, int rb, int n, int nmax, double s_r,
                                           int R, bool ex, bool real, int m, double eps,
                                           unsigned long long *err, unsigned int *fallbacks) {
    constexpr int RB = 16, LDV = 18;
    const int lane = lane_id(), r = lane & 15;
    const double *vrow = vtv_s + r * LDV;
    double s_all[RB];
    group_gather<RB>(s_r, buf, r, s_all);
    double sh;
    {
        double q4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int z = 0; z < RB; ++z) q4[z & 3] = fma(vtv_s[z * LDV + z] * s_all[z], s_all[z], q4[z & 3]);
        sh = eps * ((q4[0] + q4[1]) + (q4[2] + q4[3])) / R;
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
        if (need && r == 0) atomicAdd(fallbacks, 1u);
        const bool okLU = lu_fallback_seq<RB>(a, lu, piv, r, R, need);
        if (need && r == 0 && !okLU) report_error(err, m, DASH_E_SINGULAR);
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
            u = neg_dot4<RB>(a, xrow_v, RB) * im;
            if (!(r < R)) u = 0.0;
        }
        __syncwarp();
        if (ex && i < n) ut[(rb + i) * kSxTP + r] = u;
    }
    __syncwarp();
}

// LU fallback of the S-row system for the groups with `need` (cold path):
// returns w_r (0 for padded lanes), reports a singular / non-finite system.
// LU fallback of the S-row system (cold path; the caller holds the CTA's LU
// scratch).  D_new row r is rebuilt from the D stage (D_old) and the slice's
// U rows in the tile, in the main path's order; returns w_r for the groups
// with `need` (0 for padded lanes) and reports a singular / non-finite system.
__device__ __noinline__ double sx_b_fallback2(const double *vtv_s, double *buf, double *lu, int *piv,
                                              const double *dstage, const double *ut, int rb, int n, double lam,
                                              bool fresh, double sh2, double cn, double wv, int R, bool need,
                                              bool real, int m, unsigned long long *err, unsigned int *fallbacks) {
    constexpr int RB = 16, LDV = 18;
    const int lane = lane_id(), r = lane & 15;
    const double *vrow = vtv_s + r * LDV;
    double gram[RB];
#pragma unroll
    for (int z = 0; z < RB; ++z) gram[z] = 0.0;
    for (int i = 0; i < n; ++i) {
        const double *urw = ut + (rb + i) * kSxTP;
        const double ur = urw[r];
#pragma unroll
        for (int z = 0; z < RB; ++z) gram[z] = fma(ur, urw[z], gram[z]);
    }
    const double dg2 = real ? sh2 : 1.0;
    double a[RB];
#pragma unroll
    for (int z = 0; z < RB; ++z) {
        const double dn = real ? lam * ((fresh || z >= R) ? 0.0 : dstage[(int64_t)z * R + r]) + gram[z] : 0.0;
        a[z] = vrow[z] * dn + ((z == r) ? dg2 : 0.0);
    }
    if (need && r == 0) atomicAdd(fallbacks, 1u);
    const bool okLU = lu_fallback_seq<RB>(a, lu, piv, r, R, need);
    if (need && r == 0 && !okLU) report_error(err, m, DASH_E_SINGULAR);
    double call[RB];
    group_gather<RB>(cn, buf, r, call);
    double wv2 = 0.0;
#pragma unroll
    for (int z = 0; z < RB; ++z) wv2 = fma(-a[z], call[z], wv2);
    if (need) wv = real ? wv2 : 0.0;
    if (need && real && !isfinite(wv)) report_error(err, m, DASH_E_NONFINITE);
    return wv;
}

__global__ void __launch_bounds__(kSxThreads, 1) k_smallx(const __grid_constant__ CUtensorMap tm8,
                                                          const __grid_constant__ CUtensorMap tm16,
                                                          const __grid_constant__ CUtensorMap tm32, SxParams p) {
    using S = SxSmem;
    constexpr int RB = 16, LDV = 18;
    extern __shared__ __align__(16) double sm_raw[];
    double *sm = align1k(sm_raw);
    double *xs = sm;
    double *vt = sm + S::OFF_VT;
    double *P_s = sm + S::OFF_P;
    double *vtv_s = sm + S::OFF_VTV;
    double *slots = sm + S::OFF_SLOT;
    double *metas = sm + S::OFF_META;
    double *lu = sm + S::OFF_LU;
    int *piv = reinterpret_cast<int *>(lu + 16 * 17);
    int *lu_lock = reinterpret_cast<int *>(lu + 16 * 17 + 8);
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + S::OFF_BAR);
    uint64_t *full = bar, *empty = bar + kSxNST;
    uint64_t *uready = empty + kSxNST, *sfree = uready + kSxSlots;
    uint64_t *mready = sfree + kSxSlots, *mfree = mready + kSxNM;
    const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
    const int J = p.J, R = p.R;
    const int JS = (J + 15) / 16;

    pdl_wait();     // units, vtv (planner), previous pass / update complete
    pdl_trigger();  // k_bigx_pre may fill SMs as this kernel's CTAs retire

    if (tid == 0) {
        prefetch_map(&tm8);
        prefetch_map(&tm16);
        prefetch_map(&tm32);
        for (int s = 0; s < kSxNST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kSxMW);
        }
        for (int s = 0; s < kSxSlots; ++s) {
            mbar_init(&uready[s], kSxMW);
            mbar_init(&sfree[s], kSxSW);
        }
        for (int s = 0; s < kSxNM; ++s) {
            mbar_init(&mready[s], 1);
            mbar_init(&mfree[s], kSxMW + kSxSW);
        }
        *lu_lock = 0;
        fence_mbar_init();
    }
    // ring zeroed once: rows past a unit's boxes are stale but always finite
    for (int i = tid; i < kSxNST * S::SD; i += blockDim.x) xs[i] = 0.0;
    for (int i = tid; i < kSxNM * S::META; i += blockDim.x) metas[i] = 0.0;
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
    if (w == 0) sx_inverse_vtv(vtv_s, P_s, sm + S::OFF_SW, R, p.sweep_only);
    __syncthreads();
    const double pnorm = P_s[256];
    const bool pok = P_s[257] != 0.0;

    const int U = __ldcg(p.nunits);
    const int G = gridDim.x;
    const int u0 = (int)((int64_t)U * blockIdx.x / G), u1 = (int)((int64_t)U * (blockIdx.x + 1) / G);
    const int nmine = u1 - u0;
    const int *units = p.units + (int64_t)u0 * kSxRec;
    // item sequence of the ring (producer and math warps alike):
    // for v = 0 .. nmine + kSxLook - 1: XV(v) if v < nmine, then F(v - kSxLook) if v >= kSxLook

    if (w == kSxMW + kSxSW) {  // ---------------- TMA warp: X rows of each unit into the ring
        if (lane == 0 && nmine > 0) {
            int4 dn = __ldcg(reinterpret_cast<const int4 *>(units));
            for (int v = 0; v < nmine; ++v) {
                const int4 d = dn;
                if (v + 1 < nmine) dn = __ldcg(reinterpret_cast<const int4 *>(units + (int64_t)(v + 1) * kSxRec));
                const int st = v % kSxNST;
                if (v >= kSxNST) mbar_wait_sleep(&empty[st], (uint32_t)(((v / kSxNST) - 1) & 1));
                // boxes of 32 / 16 / 8 rows covering ceil(span / 8) row blocks of 8
                const int nb = (d.w + 7) >> 3;
                const int rows = nb == 4 ? 32 : nb == 3 ? 24 : nb * 8;
                mbar_arrive_expect_tx(&full[st], (uint32_t)(JS * rows) * 128u);
                double *dst = xs + st * S::SD;
                for (int s = 0; s < JS; ++s) {
                    if (nb == 4) {
                        tma_load_2d(dst + s * 512, &tm32, 16 * s, d.z, &full[st]);
                    } else {
                        if (nb >= 2) tma_load_2d(dst + s * 512, &tm16, 16 * s, d.z, &full[st]);
                        if (nb != 2) tma_load_2d(dst + s * 512 + (nb == 3 ? 256 : 0), &tm8, 16 * s,
                                                 d.z + (nb == 3 ? 16 : 0), &full[st]);
                    }
                }
                SX_T(v, 0);
            }
        }
        return;
    }
    if (w == kSxMW + kSxSW + 1) {  // ---------------- metadata warp
        // unit record u: lane l holds ints 2l, 2l+1 (one coalesced load per unit, issued a unit ahead)
        auto load_rec = [&](int u) -> int2 {
            return lane < kSxRec / 2 ? __ldcg(reinterpret_cast<const int2 *>(units + (int64_t)u * kSxRec) + lane)
                                     : make_int2(0, 0);
        };
        auto rec_int = [&](int2 rv, int i) -> int {  // int i of the record (warp-wide)
            const int2 x = make_int2(__shfl_sync(FULL_MASK, rv.x, i >> 1), __shfl_sync(FULL_MASK, rv.y, i >> 1));
            return (i & 1) ? x.y : x.x;
        };
        // metadata of unit u -> meta slot u % kSxNM: the record, the slices' W rows (1.0
        // for a new slice's pass-0 bootstrap) and ridge shifts sh = eps mean(vtv_rr s_r^2),
        // lane = slice; plus the unit-wide "second Neumann term needed" flag (k_slices3's test)
        auto stage = [&](int u, int2 rv) {
            const int ms = u % kSxNM, use = u / kSxNM;
            double *mt = metas + ms * S::META;
            int *mi = reinterpret_cast<int *>(mt);
            double *mw = mt + S::MHDR;
            const int q = rec_int(rv, 1);
            const bool act = lane < q;
            const int wr = rec_int(rv, 4 + kSxSlices + 1 + (lane & 15));
            const int fw = rec_int(rv, 4 + 2 * kSxSlices + 1 + ((lane & 15) >> 2));
            const bool boot = act && ((fw >> (8 * (lane & 3))) & 0xff) != 0 && p.pass == 0;
            double sv[16];
#pragma unroll
            for (int z = 0; z < 8; ++z) {
                double2 w2 = make_double2(0.0, 0.0);
                if (act && 2 * z < R) w2 = boot ? make_double2(1.0, 1.0)
                                                : __ldcg(reinterpret_cast<const double2 *>(p.W + (int64_t)wr * R) + z);
                sv[2 * z] = w2.x;
                sv[2 * z + 1] = (2 * z + 1 < R) ? w2.y : 0.0;
            }
            double q4[4] = {0.0, 0.0, 0.0, 0.0};
            double smin = INFINITY;
#pragma unroll
            for (int z = 0; z < 16; ++z) {
                q4[z & 3] = fma(vtv_s[z * LDV + z] * sv[z], sv[z], q4[z & 3]);
                if (z < R) smin = fmin(smin, sv[z] * sv[z]);
            }
            const double sh = p.eps * ((q4[0] + q4[1]) + (q4[2] + q4[3])) / R;
            const double rho = sh * (1.0 / smin) * pnorm;  // s_r = 0 -> inf; non-finite s -> non-finite sh
            const bool need2 = act && pok && rho <= kS3Neumann && !(rho <= kS3Neumann1);
            const int any2 = __any_sync(FULL_MASK, need2) ? 1 : 0;
            if (use >= 1) mbar_wait_sleep(&mfree[ms], (uint32_t)((use - 1) & 1));
            if (lane < kSxRec / 2) {
                int2 hv = rv;
                if (lane == (4 + 2 * kSxSlices + 1 + 4) / 2) hv.y = any2;  // int 41
                reinterpret_cast<int2 *>(mi)[lane] = hv;
            }
            if (act) {
#pragma unroll
                for (int z = 0; z < 8; ++z)
                    *reinterpret_cast<double2 *>(mw + lane * 16 + 2 * z) = make_double2(sv[2 * z], sv[2 * z + 1]);
                mt[S::MSH + lane] = sh;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&mready[ms]);
        };
        if (nmine > 0) {
            int2 rnext = load_rec(0);
            for (int v = 0; v < nmine; ++v) {
                const int2 rcur = rnext;
                if (v + 1 < nmine) rnext = load_rec(v + 1);
                stage(v, rcur);
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
        int64_t item = 0;
        for (int v = 0; v < nmine; ++v) {
            {  // ---- XV(v), Y, the Neumann U of this warp's 8 rows
                const int u = v, slot = u % kSxSlots, use = u / kSxSlots, ms = u % kSxNM;
                const int st = (int)(item % kSxNST);
                mbar_wait_sleep(&full[st], (uint32_t)((item / kSxNST) & 1));
                ++item;
                if (mb == 0 && lane == 0) SX_T(u, 2);
                SX_M(u, 0);
                const double *xt = xs + st * S::SD;
                double xa[2][2][2];
#pragma unroll
                for (int nb = 0; nb < 2; ++nb)
#pragma unroll
                    for (int c = 0; c < 2; ++c) xa[nb][c][0] = xa[nb][c][1] = 0.0;
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
                                dmma884(xa[nb][0], a.x, b.x);
                                dmma884(xa[nb][1], a.y, b.y);
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
                    for (int e = 0; e < 2; ++e) xv[nb][e] = xa[nb][0][e] + xa[nb][1][e];
                SX_M(u, 1);
                // the row's slice and its W row (staged by the producer)
                mbar_wait_sleep(&mready[ms], (uint32_t)((u / kSxNM) & 1));
                SX_M(u, 2);
                const double *mt = metas + ms * S::META;
                const int *mi = reinterpret_cast<const int *>(mt);
                const int q = mi[1], span = mi[3];
                int j = 0;
                for (int k = 1; k < q; ++k) j += (mi[4 + k] <= xrow) ? 1 : 0;
                const bool valid = xrow < span;
                const double *sw = mt + S::MHDR + j * 16;
                const double sh = valid ? mt[S::MSH + j] : 0.0;
                const int any2 = mi[4 + 2 * kSxSlices + 1 + 4];
                double dd[2][2], si[2][2];
#pragma unroll
                for (int nb = 0; nb < 2; ++nb) {
                    const double2 s2 = *reinterpret_cast<const double2 *>(sw + 8 * nb + 2 * t);
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int c = 8 * nb + 2 * t + e;
                        const double is = (valid && c < R) ? rcp_nr(e ? s2.y : s2.x) : 0.0;
                        si[nb][e] = is;
                        dd[nb][e] = sh * is * is;
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&mfree[ms]);  // last read of the metadata slot
                SX_M(u, 3);
                // Y = XV P: A fragment of K step kk = this lane's XV value xv[kk >> 1][kk & 1]
                double ya[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
#pragma unroll
                    for (int nb = 0; nb < 2; ++nb) dmma884(ya[nb], xv[kk >> 1][kk & 1], pf[kk][nb]);
                double c1[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
#pragma unroll
                    for (int nb = 0; nb < 2; ++nb)
                        dmma884(c1[nb], ya[kk >> 1][kk & 1] * dd[kk >> 1][kk & 1], pf[kk][nb]);  // (Y o d) P
                double c2[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
                if (any2) {  // unit-uniform
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
#pragma unroll
                        for (int nb = 0; nb < 2; ++nb)
                            dmma884(c2[nb], c1[kk >> 1][kk & 1] * dd[kk >> 1][kk & 1], pf[kk][nb]);
                }
                SX_M(u, 4);
                double *sl = slots + slot * S::SLOT;
                double *xvt = sl, *ut = sl + S::TILE;
                if (use >= 1) mbar_wait_sleep(&sfree[slot], (uint32_t)((use - 1) & 1));  // solvers done with u - kSxSlots
                SX_M(u, 5);
#pragma unroll
                for (int nb = 0; nb < 2; ++nb) {
                    *reinterpret_cast<double2 *>(xvt + xrow * kSxTP + 8 * nb + 2 * t) = make_double2(xv[nb][0], xv[nb][1]);
                    double u2[2];
#pragma unroll
                    for (int e = 0; e < 2; ++e) u2[e] = valid ? ((ya[nb][e] - c1[nb][e]) + c2[nb][e]) * si[nb][e] : 0.0;
                    *reinterpret_cast<double2 *>(ut + xrow * kSxTP + 8 * nb + 2 * t) = make_double2(u2[0], u2[1]);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&uready[slot]);
                if (mb == 0 && lane == 0) SX_T(u, 3);
                SX_M(u, 6);
            }
        }
        return;
    }
    // ---------------- solver warps: slice pairs round-robin over the unit sequence
    const int ws = w - kSxMW;
    const int r = lane & 15, gl = lane >> 4;
    double *buf = sm + S::OFF_SW + ws * S::SWS + gl * 18;
    double *dstage = sm + S::OFF_SW + ws * S::SWS + 36 + gl * 256;  // the pair's D block, column r at [z * 16 + r]
    const double *vrow = vtv_s + r * LDV;
    int pc = 0;  // pairs of the units before this one
#ifdef DASH_SX_TRACE
    long long t_busy = 0, t_wait = 0, n_pairs = 0, t_start = clock64();
#endif
    for (int u = 0; u < nmine; ++u) {
        const int slot = u % kSxSlots, use = u / kSxSlots, ms = u % kSxNM;
        mbar_wait_sleep(&mready[ms], (uint32_t)((u / kSxNM) & 1));
        const double *mt = metas + ms * S::META;
        const int *mi = reinterpret_cast<const int *>(mt);
        const uint8_t *mf = reinterpret_cast<const uint8_t *>(mi + 4 + 2 * kSxSlices + 1);
        const int m0 = mi[0], q = mi[1], a0 = mi[2];
        const int np = (q + 1) >> 1;
        const int k0 = ((ws - pc) % kSxSW + kSxSW) % kSxSW;  // my first pair of this unit
        pc += np;
        bool waited = false;
        for (int k = k0; k < np; k += kSxSW) {
#ifdef DASH_SX_TRACE
            const long long tp0 = clock64();
            ++n_pairs;
#endif
            SX_P(0);
            const int j = 2 * k + gl;
            const bool act = j < q;
            const bool real = act && r < R;
            const int m = m0 + (act ? j : 0);
            const int rb = act ? mi[4 + j] : 0;
            const int n = act ? mi[4 + j + 1] - rb : 0;
            const int64_t rg = (int64_t)a0 + rb;
            const int wrow = act ? mi[4 + kSxSlices + 1 + j] : 0;
            const bool fresh = act && mf[j] != 0;
            const double s_r = real ? mt[S::MHDR + j * 16 + r] : 0.0;
            // state (latency overlaps the rows loop): c_old, D column r
            // state: D block -> dstage (cp.async, waited for after the rows loop), c_old
            const bool ld = real && !fresh;
            double cold = 0.0;
            if (ld) {
                const double *dcol = p.D + (int64_t)wrow * R * R + r;
                for (int z = 0; z < R; ++z) cp_async8(dstage + z * 16 + r, dcol + (int64_t)z * R);
                cold = __ldcg(p.C + (int64_t)wrow * R + r);
            }
            if (!waited) {
                mbar_wait_sleep(&uready[slot], (uint32_t)(use & 1));
                waited = true;
                if (lane == 0) SX_T(u, 5);
            }
            SX_P(1);
            double *xvt = slots + slot * S::SLOT, *ut = xvt + S::TILE;
            int nmax = n;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) nmax = max(nmax, __shfl_xor_sync(FULL_MASK, nmax, off));
            // the Neumann test again (the math warps applied it per row): exact path otherwise
            bool fast;
            {
                double s_all[RB];
                group_gather<RB>(s_r, buf, r, s_all);
                double q4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                for (int z = 0; z < RB; ++z) q4[z & 3] = fma(vtv_s[z * LDV + z] * s_all[z], s_all[z], q4[z & 3]);
                const double sh = p.eps * ((q4[0] + q4[1]) + (q4[2] + q4[3])) / R;
                double qm = 0.0;
                if (real) {
                    const double is = rcp_nr(s_r);
                    const double qz = is * is;
                    qm = (s_r != 0.0 && isfinite(qz)) ? qz : INFINITY;
                }
#pragma unroll
                for (int off = 8; off > 0; off >>= 1) qm = fmax(qm, __shfl_xor_sync(FULL_MASK, qm, off));
                const double rho = sh * qm * pnorm;
                fast = act && pok && rho <= kS3Neumann;
            }
            SX_P(2);
            if (__any_sync(FULL_MASK, act && !fast)) {  // rare: exact A solve; serialised LU scratch
                if (lane == 0)
                    while (atomicCAS(lu_lock, 0, 1) != 0) __nanosleep(64);
                __syncwarp();
                sx_exact_rows(vtv_s, buf, lu, piv, xvt, ut, rb, n, nmax, s_r, R, act && !fast, real, m, p.eps,
                              p.err, p.fallbacks);
                __syncwarp();
                if (lane == 0) atomicExch(lu_lock, 0);
            }
            SX_P(3);
            // ---- rows: U -> U_out, c, gram (_kernels.py:98-115)
            double c = 0.0, gram[RB];
#pragma unroll
            for (int z = 0; z < RB; ++z) gram[z] = 0.0;
            for (int i = 0; i < n; ++i) {
                const double *urw = ut + (rb + i) * kSxTP;
                double ua[RB];
#pragma unroll
                for (int z = 0; z < RB / 2; ++z) {
                    const double2 t2 = *reinterpret_cast<const double2 *>(urw + 2 * z);
                    ua[2 * z] = t2.x;
                    ua[2 * z + 1] = t2.y;
                }
                const double ur = urw[r];
#pragma unroll
                for (int z = 0; z < RB; ++z) gram[z] = fma(ur, ua[z], gram[z]);
                if (real) {
                    c = fma(xvt[(rb + i) * kSxTP + r], ur, c);
                    p.U[(rg + i) * R + r] = ur;
                }
            }
            // ---- c, D accumulation and the S-row system (_kernels.py:103-135)
            SX_P(4);
            const double cn = real ? p.lam * cold + c : 0.0;
            double a[RB];
            double drr = 0.0;
            cp_async_wait();
            __syncwarp();
#pragma unroll
            for (int z = 0; z < RB; ++z) {
                const double dn = real ? p.lam * ((ld && z < R) ? dstage[z * 16 + r] : 0.0) + gram[z] : 0.0;
                a[z] = dn;  // D_new row r (rows / columns >= R are 0)
                if (z == r) drr = dn;
            }
            SX_P(5);
            if (real && p.final_pass) {
                p.C[(int64_t)wrow * R + r] = cn;
#pragma unroll
                for (int z = 0; z < RB; ++z)
                    if (z < R) p.D[(int64_t)wrow * R * R + (int64_t)z * R + r] = a[z];
            }
            SX_P(6);
            double sh2;
            {
                double vdd[RB];
                group_gather<RB>(real ? vrow[r] * drr : 0.0, buf, r, vdd);
                double dsum = 0.0;
#pragma unroll
                for (int z = 0; z < RB; ++z) dsum += vdd[z];
                sh2 = p.eps * dsum / R;
            }
            const double dg2 = real ? sh2 : 1.0;
#pragma unroll
            for (int z = 0; z < RB; ++z) a[z] = vrow[z] * a[z] + ((z == r) ? dg2 : 0.0);
            SX_P(7);
            double wv;
            const bool okB = gj_solve<RB>(a, cn, buf, r, wv);
            SX_P(8);
            if (!real) wv = 0.0;
            bool gok = okB && isfinite(wv);
            {
                const unsigned bal = __ballot_sync(FULL_MASK, !gok);
                gok = (bal & (0xffffu << (gl * 16))) == 0;
            }
            if (__any_sync(FULL_MASK, !gok && act)) {  // rare: LU (the reference's numpy fallback)
                if (lane == 0)
                    while (atomicCAS(lu_lock, 0, 1) != 0) __nanosleep(64);
                __syncwarp();
                wv = sx_b_fallback2(vtv_s, buf, lu, piv, p.D + (int64_t)wrow * R * R, ut, rb, n, p.lam, fresh,
                                    sh2, cn, wv, R, !gok && act, real, m, p.err, p.fallbacks);
                __syncwarp();
                if (lane == 0) atomicExch(lu_lock, 0);
            }
            SX_P(9);
            if (real) {
                p.W[(int64_t)wrow * R + r] = wv;
                for (int i = 0; i < n; ++i) p.US[(rg + i) * R + r] = ut[(rb + i) * kSxTP + r] * wv;
            }
            SX_P(10);
#ifdef DASH_SX_TRACE
            t_busy += clock64() - tp0;
#endif
        }
        if (!waited) mbar_wait_sleep(&uready[slot], (uint32_t)(use & 1));
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(&mfree[ms]);
            mbar_arrive(&sfree[slot]);
        }
        if (lane == 0 && k0 < np) SX_T(u, 6);
    }
#ifdef DASH_SX_TRACE
    if (blockIdx.x == 0 && lane == 0) {
        g_sxtrace2[512 + ws * 4 + 0] = t_busy;
        g_sxtrace2[512 + ws * 4 + 1] = n_pairs;
        g_sxtrace2[512 + ws * 4 + 2] = clock64() - t_start;
    }
#endif
}

int launch_smallx(dash_ctx *ctx, cudaStream_t st, const CUtensorMap &m8, const CUtensorMap &m16,
                  const CUtensorMap &m32, const SxParams &sp, int grid) {
    const size_t smem = SxSmem::bytes();
    ensure_smem_attr(k_smallx, smem);
    return launch_k(pdl_site("smallx"), k_smallx, grid, kSxThreads, smem, st, m8, m16, m32, sp);
}
