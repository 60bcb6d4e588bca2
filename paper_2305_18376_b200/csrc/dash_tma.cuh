// TMA-tensor streaming GEMMs (R bucket 16): the same two contractions as
// dash_stream.cuh, but each 32-row tile arrives as ceil(J/16) tensor copies
// (cp.async.bulk.tensor.2d, box 16 doubles x 32 rows, 128-byte swizzle)
// instead of 32 one-row bulk copies -- the per-copy cost of small bulk copies
// capped the v2 kernels at ~4.9 TB/s (tools/bulk_probe.cu: 6.9 TB/s with one
// large copy per tile).
//
// Fragment loads are LDS.128 pairs on the swizzled layout:
//   k_xv3    XV = X V: each lane reads X[row][2c, 2c+1] and feeds two DMMA
//            k-steps whose K orders are the even / odd columns of an 8-column
//            group; V is staged transposed (Vt[n][k]) so the matching B pair is
//            one LDS.128 too.
//   k_fgemm3 F = X^T US: the M (=j) and N (=r) dimensions are split into even
//            / odd halves, so one LDS.128 of X and one of US feed a 2x2 block of
//            DMMA tiles; the permutation is undone when the slot is written.
// With the 128B swizzle (16-byte chunk c of row r stored at c ^ (r & 7)) all
// these reads are bank-conflict-free.  Rows past N are zero-filled by TMA.
// (included inside dash_update.cu's anonymous namespace)
#pragma once

#include <cuda.h>

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int r0, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(c0), "r"(r0), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap *map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

// double offset of the 16-byte chunk `c` (0..7) of row `r` inside a swizzled 32x16 box
__device__ __forceinline__ int swz(int r, int c) { return r * 16 + ((c ^ (r & 7)) << 1); }

// LDS.128 is serviced per quarter-warp (8 lanes = fragment rows g = 2q, 2q+1):
// mapping fragment index g to perm(g) = (g&1)*4 + g/2 makes the two rows of a
// quarter-warp XOR-swizzle into disjoint chunk halves -> conflict-free.  The
// permutation is undone when results are written.
__device__ __forceinline__ int qperm(int g) { return ((g & 1) << 2) | (g >> 1); }

// Tile-visit mask for 32 consecutive local tiles i0 .. i0+31 of this CTA
// (tile = blockIdx.x + i * gridDim.x): one coalesced flag load per lane and a
// ballot, so the skip test costs one global round trip per 32 tiles.
__device__ __forceinline__ unsigned visit_mask(const uint32_t *tflag, uint32_t tgen, int64_t i0, int64_t mine) {
    const int64_t i = i0 + lane_id();
    const bool v = i < mine && (tflag == nullptr || tflag[blockIdx.x + i * gridDim.x] == tgen);
    return __ballot_sync(FULL_MASK, v);
}

struct TmaSmem {
    static __host__ __device__ int strips(int J) { return (J + 15) / 16; }
    static __host__ __device__ int vtp(int J) { return strips(J) * 16 + 8; }  // Vt pitch (== 8 mod 16)
    static __host__ __device__ size_t stage_doubles(int J) { return (size_t)strips(J) * 512; }
    static __host__ __device__ size_t xv_bytes(int J) {
        return 1024 + sizeof(double) * (kStages * stage_doubles(J) + 16 * (size_t)vtp(J)) + 16 * kStages;
    }
    static __host__ __device__ size_t f_bytes(int J) {
        return 1024 + sizeof(double) * (kStages * (stage_doubles(J) + 512)) + 16 * kStages;
    }
};

// 1024-byte alignment for the swizzled boxes; pointer arithmetic (not an integer
// round trip) so the compiler keeps the shared address space and emits LDS.
__device__ __forceinline__ double *align1k(double *p) {
    return p + (((1024u - (smem_u32(p) & 1023u)) & 1023u) >> 3);
}

// Pass prologue fused into the XV kernel (no separate launch): CTA 0 forms
// vtv = V^T V from its staged V^T, and all CTAs share the F / G snapshot and
// v_used copies (what k_prologue does on the other paths).
struct FusedPrologue {
    double *vtv;
    const double *F, *G;
    double *F_snap, *G_snap, *v_used;
    int snap, last;
};

// tflag (optional): visit only tiles with tflag[tile] == tgen (the small-slice
// tiles when big slices take the fused path); producer and consumers skip the
// same tiles, the ring advances only on visited ones.
__global__ void __launch_bounds__(kCW * 32 + 32, 1) k_xv3(const __grid_constant__ CUtensorMap tmX, int64_t N, int J,
                                                          const double *__restrict__ V, int R, double *__restrict__ XV,
                                                          FusedPrologue pro, const uint32_t *__restrict__ tflag,
                                                          uint32_t tgen) {
    extern __shared__ __align__(16) double sm_raw[];
    double *sm = align1k(sm_raw);
    const int JS = TmaSmem::strips(J), VTP = TmaSmem::vtp(J);
    const size_t SD = TmaSmem::stage_doubles(J);
    double *xs = sm;                               // kStages x JS x 512 (swizzled 32x16 boxes)
    double *vt = xs + kStages * SD;                // 16 x VTP: vt[n][k] = V[k][n]
    uint64_t *full = reinterpret_cast<uint64_t *>(vt + 16 * VTP);
    uint64_t *empty = full + kStages;
    const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
    const int g = lane >> 2, t = lane & 3;
    // PDL: needs nothing from the plan kernels before it (X, V are final once
    // the update's first, normally launched kernel has started); waits only
    // at exit so that its completion implies theirs.
    pdl_trigger();
    if (tid == 0) {
        prefetch_map(&tmX);
        for (int s2 = 0; s2 < kStages; ++s2) {
            mbar_init(&full[s2], 1);
            mbar_init(&empty[s2], kCW);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int64_t ntiles = (N + kTR - 1) / kTR;
    const int64_t mine = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    if (w == kCW) {
        for (int64_t i0 = 0, k = 0; i0 < mine; i0 += 32) {
            unsigned vm = visit_mask(tflag, tgen, i0, mine);
            if (lane == 0) {
                while (vm) {
                    const int b = __ffs(vm) - 1;
                    vm &= vm - 1;
                    const int64_t tile = blockIdx.x + (i0 + b) * gridDim.x;
                    const int st = (int)(k % kStages);
                    if (k >= kStages) mbar_wait(&empty[st], (uint32_t)(((k / kStages) - 1) & 1));
                    ++k;
                    const int r0 = (int)(tile * kTR);
                    mbar_arrive_expect_tx(&full[st], (uint32_t)JS * 4096u);
                    for (int s = 0; s < JS; ++s) tma_load_2d(xs + st * SD + s * 512, &tmX, 16 * s, r0, &full[st]);
                }
            }
            __syncwarp();
        }
        pdl_wait();
        return;
    }
    // consumers: V^T staging and the fused prologue overlap the producer's first loads
    for (int i = tid; i < 16 * VTP; i += kCW * 32) {
        const int nn = i / VTP, k = i % VTP;
        vt[i] = (nn < R && k < J) ? V[k * R + nn] : 0.0;
    }
    compute_bar();
    {
        const int gt = blockIdx.x * (kCW * 32) + tid, nt = gridDim.x * (kCW * 32);
        if (pro.snap) {
            for (int i = gt; i < J * R; i += nt) pro.F_snap[i] = pro.F[i];
            for (int i = gt; i < R * R; i += nt) pro.G_snap[i] = pro.G[i];
        }
        if (pro.last)
            for (int i = gt; i < J * R; i += nt) pro.v_used[i] = V[i];
        if (blockIdx.x == 0 && tid < R * R) {  // vtv[r][z] = sum_k V[k][r] V[k][z], 4 chains
            const double *a = vt + (tid / R) * VTP, *b = vt + (tid % R) * VTP;
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            for (int k = 0; k < J; k += 4)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[q] = fma(a[k + q], b[k + q], acc[q]);  // vt padded to 16
            pro.vtv[tid] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
        }
    }
    const int mb = w & 3, nb = w >> 2;  // 8-row block, 8-column block of the 32 x 16 output tile
    const double *vrow = vt + (8 * nb + g) * VTP + 2 * t;
    const int row = 8 * mb + qperm(g);  // tile row of this lane's A fragment and output
    unsigned vm = 0;
    for (int64_t i = 0, k = -1; i < mine; ++i) {
        if ((i & 31) == 0) vm = visit_mask(tflag, tgen, i, mine);
        if (!((vm >> (i & 31)) & 1u)) continue;
        ++k;
        const int st = (int)(k % kStages);
        mbar_wait(&full[st], (uint32_t)((k / kStages) & 1));
        const double *xt = xs + st * SD;
        double acc[2] = {0.0, 0.0}, acc2[2] = {0.0, 0.0};
        for (int s = 0; s < JS; ++s) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {  // 8-column group h of the strip
                const double2 a = *reinterpret_cast<const double2 *>(xt + s * 512 + swz(row, 4 * h + t));
                const double2 b = *reinterpret_cast<const double2 *>(vrow + 16 * s + 8 * h);
                dmma884(acc, a.x, b.x);   // k-order: even columns of the group
                dmma884(acc2, a.y, b.y);  // odd columns
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        const int64_t grow = (blockIdx.x + i * gridDim.x) * kTR + row;
        if (grow < N) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int col = 8 * nb + 2 * t + e;
                if (col < R) XV[grow * R + col] = acc[e] + acc2[e];
            }
        }
    }
    pdl_wait();
}

// F slot = sum over this CTA's tiles of X^T US.  Warp w owns J-strips w, w+8, ...
// (MAXS strips); per strip a 2x2 block of 8x8 DMMA tiles (even/odd j x even/odd r).
template <int MAXS>
__global__ void __launch_bounds__(kCW * 32 + 32, 1) k_fgemm3(const __grid_constant__ CUtensorMap tmX,
                                                             const __grid_constant__ CUtensorMap tmU, int64_t N, int J,
                                                             int R, double *__restrict__ F_slots,
                                                             const uint32_t *__restrict__ tflag, uint32_t tgen,
                                                             double *__restrict__ G_slots = nullptr) {
    extern __shared__ __align__(16) double sm_raw[];
    double *sm = align1k(sm_raw);
    const int JS = TmaSmem::strips(J);
    const size_t SD = TmaSmem::stage_doubles(J) + 512;  // X boxes + the US box
    double *xs = sm;
    uint64_t *full = reinterpret_cast<uint64_t *>(xs + kStages * SD);
    uint64_t *empty = full + kStages;
    const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
    const int g = lane >> 2, t = lane & 3;
    if (tid == 0) {
        prefetch_map(&tmX);
        prefetch_map(&tmU);
        for (int s2 = 0; s2 < kStages; ++s2) {
            mbar_init(&full[s2], 1);
            mbar_init(&empty[s2], kCW);
        }
        fence_mbar_init();
    }
    __syncthreads();
    pdl_wait();     // US from the slice kernels
    pdl_trigger();  // only now: a successor may rely on everything before this kernel
    const int64_t ntiles = (N + kTR - 1) / kTR;
    const int64_t mine = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    if (w == kCW) {
        for (int64_t i0 = 0, k = 0; i0 < mine; i0 += 32) {
            unsigned vm = visit_mask(tflag, tgen, i0, mine);
            if (lane == 0) {
                while (vm) {
                    const int b = __ffs(vm) - 1;
                    vm &= vm - 1;
                    const int64_t tile = blockIdx.x + (i0 + b) * gridDim.x;
                    const int st = (int)(k % kStages);
                    if (k >= kStages) mbar_wait(&empty[st], (uint32_t)(((k / kStages) - 1) & 1));
                    ++k;
                    const int r0 = (int)(tile * kTR);
                    mbar_arrive_expect_tx(&full[st], (uint32_t)(JS + 1) * 4096u);
                    for (int s = 0; s < JS; ++s) tma_load_2d(xs + st * SD + s * 512, &tmX, 16 * s, r0, &full[st]);
                    tma_load_2d(xs + st * SD + JS * 512, &tmU, 0, r0, &full[st]);
                }
            }
            __syncwarp();
        }
        return;
    }
    const int pg = qperm(g);  // j pair (A) and r pair (B) of this lane: 2 pg, 2 pg + 1
    double acc[MAXS][4][2];
#pragma unroll
    for (int q = 0; q < MAXS; ++q)
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[q][k][0] = acc[q][k][1] = 0.0;
    // optional G = sum US^T US (the fused small-slice path: sum_k gram_k o w_k w_k^T
    // over the small slices), block (w >> 1, w & 1) on warps 0..3
    const bool gw = G_slots != nullptr && w < 4;
    const int gmi = w >> 1, gni = w & 1;
    double gacc[2] = {0.0, 0.0};
    unsigned vm = 0;
    for (int64_t i = 0, k = -1; i < mine; ++i) {
        if ((i & 31) == 0) vm = visit_mask(tflag, tgen, i, mine);
        if (!((vm >> (i & 31)) & 1u)) continue;
        ++k;
        const int st = (int)(k % kStages);
        mbar_wait(&full[st], (uint32_t)((k / kStages) & 1));
        const double *xt = xs + st * SD;
        const double *ut = xt + JS * 512;
#pragma unroll
        for (int kk = 0; kk < kTR / 4; ++kk) {
            const int row = 4 * kk + t;
            if (gw) {
                const int ca = 8 * gmi + g, cb = 8 * gni + g;
                dmma884(gacc, ut[swz(row, ca >> 1) + (ca & 1)], ut[swz(row, cb >> 1) + (cb & 1)]);
            }
            const double2 b = *reinterpret_cast<const double2 *>(ut + swz(row, pg));  // US[row][2pg], [2pg+1]
#pragma unroll
            for (int q = 0; q < MAXS; ++q) {
                const int s = w + kCW * q;
                if (s < JS) {
                    const double2 a = *reinterpret_cast<const double2 *>(xt + s * 512 + swz(row, pg));
                    dmma884(acc[q][0], a.x, b.x);  // even j, even r
                    dmma884(acc[q][1], a.x, b.y);  // even j, odd r
                    dmma884(acc[q][2], a.y, b.x);  // odd j, even r
                    dmma884(acc[q][3], a.y, b.y);  // odd j, odd r
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
    }
    double *slot = F_slots + (int64_t)blockIdx.x * J * R;
#pragma unroll
    for (int q = 0; q < MAXS; ++q) {
        const int s = w + kCW * q;
        if (s < JS) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int j = 16 * s + 2 * pg + (k >> 1);
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int r = 2 * qperm(2 * t + e) + (k & 1);
                    if (j < J && r < R) slot[j * R + r] = acc[q][k][e];
                }
            }
        }
    }
    if (gw) {
        double *gs = G_slots + (int64_t)blockIdx.x * R * R;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int a = 8 * gmi + g, b = 8 * gni + 2 * t + e;
            if (a < R && b < R) gs[a * R + b] = gacc[e];
        }
    }
}
