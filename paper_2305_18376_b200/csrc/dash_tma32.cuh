// FP32 data mode of the two TMA streaming GEMMs (R bucket 16): X arrives as
// FLOAT32 tensor boxes (32 floats x 32 rows = one 128-byte swizzled row per
// tile row, cp.async.bulk.tensor.2d), half the HBM bytes of the FP64 path.
// Products and sums stay in FP64 on the DMMA tensor cores: each float is
// widened in registers (F2F.F64.F32) before it enters a fragment, so the only
// FP32 rounding is the caller's rounding of X itself (and of U_new on output).
//
//   k_xv3f    XV = X V: one LDS.128 of a swizzled 16-byte chunk gives a lane 4
//             consecutive columns of its fragment row -> four DMMA k-steps
//             (separate accumulator chains); V^T is staged FP64 with a pitch
//             == 2 (mod 16) doubles so the two matching LDS.128 of B are
//             conflict-free across a quarter-warp.
//   k_fgemm3f F_slot = X^T US: a lane's float4 of X covers 4 consecutive j
//             (4 DMMA j-tiles) and its double2 of US 2 consecutive r (2 r-tiles)
//             -> a 4 x 2 block of tiles per LDS pair.  A tile carries half as
//             many j-strips as the FP64 box, so the 8 compute warps split the
//             rows of a tile into kRG interleaved row groups (one F slot per CTA
//             and row group, summed later in fixed order -> deterministic).
// Both keep k_xv3 / k_fgemm3's producer warp, mbarrier ring (8 stages here), qperm
// fragment permutation and fused prologue.
// (included inside dash_update.cu's anonymous namespace, after dash_tma.cuh)
#pragma once

// Ring depth: 8 stages of half-size (FP32) tiles keep the FP64 kernels' bytes
// in flight, and push the footprint past half the SM's shared memory so the
// persistent grid gets exactly one CTA per SM (two 80 KB CTAs landing on one
// SM while another still runs the predecessor cost 160 us / update).
constexpr int kStages32 = 8;

// float offset of 16-byte chunk `c` (0..7) of row `r` inside a swizzled 32x32-float box
__device__ __forceinline__ int swzf(int r, int c) { return r * 32 + ((c ^ (r & 7)) << 2); }

struct TmaSmem32 {
    static __host__ __device__ int strips(int J) { return (J + 31) / 32; }
    static __host__ __device__ int vtp(int J) { return strips(J) * 32 + 2; }  // == 2 (mod 16)
    static __host__ __device__ size_t stage_bytes(int J) { return (size_t)strips(J) * 4096; }
    static __host__ __device__ size_t xv_bytes(int J) {
        return 1024 + kStages32 * stage_bytes(J) + sizeof(double) * 16 * (size_t)vtp(J) + 16 * kStages32;
    }
    static __host__ __device__ size_t f_bytes(int J) { return 1024 + kStages32 * (stage_bytes(J) + 4096) + 16 * kStages32; }
    // row groups of k_fgemm3f: 8 compute warps = (8 / rg) strip slots x rg row groups
    static __host__ __device__ int row_groups(int J) {
        const int s = strips(J);
        return s <= 2 ? 4 : s <= 4 ? 2 : 1;
    }
};

__device__ __forceinline__ float *align1kf(float *p) {
    return p + (((1024u - (smem_u32(p) & 1023u)) & 1023u) >> 2);
}

__global__ void __launch_bounds__(kCW * 32 + 32, 1) k_xv3f(const __grid_constant__ CUtensorMap tmX, int64_t N, int J,
                                                           const double *__restrict__ V, int R, double *__restrict__ XV,
                                                           FusedPrologue pro, const uint32_t *__restrict__ tflag,
                                                           uint32_t tgen) {
    extern __shared__ __align__(16) float smf_raw[];
    float *sm = align1kf(smf_raw);
    const int JS = TmaSmem32::strips(J), VTP = TmaSmem32::vtp(J);
    const size_t SF = TmaSmem32::stage_bytes(J) / 4;  // floats per stage
    float *xs = sm;                                    // kStages32 x JS x 1024 (swizzled 32x32 boxes)
    double *vt = reinterpret_cast<double *>(xs + kStages32 * SF);  // 16 x VTP: vt[n][k] = V[k][n]
    uint64_t *full = reinterpret_cast<uint64_t *>(vt + 16 * VTP);
    uint64_t *empty = full + kStages32;
    const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
    const int g = lane >> 2, t = lane & 3;
    pdl_trigger();
    if (tid == 0) {
        prefetch_map(&tmX);
        for (int s2 = 0; s2 < kStages32; ++s2) {
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
                    const int st = (int)(k % kStages32);
                    if (k >= kStages32) mbar_wait(&empty[st], (uint32_t)(((k / kStages32) - 1) & 1));
                    ++k;
                    const int r0 = (int)(tile * kTR);
                    mbar_arrive_expect_tx(&full[st], (uint32_t)JS * 4096u);
                    for (int s = 0; s < JS; ++s) tma_load_2d(xs + st * SF + s * 1024, &tmX, 32 * s, r0, &full[st]);
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
        if (blockIdx.x == 0 && tid < R * R) {
            const double *a = vt + (tid / R) * VTP, *b = vt + (tid % R) * VTP;
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            for (int k = 0; k < J; k += 4)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[q] = fma(a[k + q], b[k + q], acc[q]);  // vt padded to 32
            pro.vtv[tid] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
        }
    }
    const int mb = w & 3, nb = w >> 2;
    const double *vrow = vt + (8 * nb + g) * VTP + 4 * t;
    const int row = 8 * mb + qperm(g);
    unsigned vm = 0;
    for (int64_t i = 0, k = -1; i < mine; ++i) {
        if ((i & 31) == 0) vm = visit_mask(tflag, tgen, i, mine);
        if (!((vm >> (i & 31)) & 1u)) continue;
        ++k;
        const int st = (int)(k % kStages32);
        mbar_wait(&full[st], (uint32_t)((k / kStages32) & 1));
        const float *xt = xs + st * SF;
        double acc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
        for (int s = 0; s < JS; ++s) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {  // columns 32 s + 16 h + 4 t + {0..3}
                const float4 a = *reinterpret_cast<const float4 *>(xt + s * 1024 + swzf(row, 4 * h + t));
                const double2 b0 = *reinterpret_cast<const double2 *>(vrow + 32 * s + 16 * h);
                const double2 b1 = *reinterpret_cast<const double2 *>(vrow + 32 * s + 16 * h + 2);
                dmma884(acc[0], (double)a.x, b0.x);
                dmma884(acc[1], (double)a.y, b0.y);
                dmma884(acc[2], (double)a.z, b1.x);
                dmma884(acc[3], (double)a.w, b1.y);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        const int64_t grow = (blockIdx.x + i * gridDim.x) * kTR + row;
        if (grow < N) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int col = 8 * nb + 2 * t + e;
                if (col < R) XV[grow * R + col] = (acc[0][e] + acc[1][e]) + (acc[2][e] + acc[3][e]);
            }
        }
    }
    pdl_wait();
}

// F slot (CTA b, row group q) at F_slots + (b * RG + q) * J * R.
__global__ void __launch_bounds__(kCW * 32 + 32, 1) k_fgemm3f(const __grid_constant__ CUtensorMap tmX,
                                                              const __grid_constant__ CUtensorMap tmU, int64_t N,
                                                              int J, int R, double *__restrict__ F_slots,
                                                              const uint32_t *__restrict__ tflag, uint32_t tgen) {
    extern __shared__ __align__(16) float smf_raw[];
    float *sm = align1kf(smf_raw);
    const int JS = TmaSmem32::strips(J), RG = TmaSmem32::row_groups(J);
    const size_t SF = (TmaSmem32::stage_bytes(J) + 4096) / 4;  // X boxes + the US box (floats)
    float *xs = sm;
    uint64_t *full = reinterpret_cast<uint64_t *>(xs + kStages32 * SF);
    uint64_t *empty = full + kStages32;
    const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
    const int g = lane >> 2, t = lane & 3;
    if (tid == 0) {
        prefetch_map(&tmX);
        prefetch_map(&tmU);
        for (int s2 = 0; s2 < kStages32; ++s2) {
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
                    const int st = (int)(k % kStages32);
                    if (k >= kStages32) mbar_wait(&empty[st], (uint32_t)(((k / kStages32) - 1) & 1));
                    ++k;
                    const int r0 = (int)(tile * kTR);
                    mbar_arrive_expect_tx(&full[st], (uint32_t)(JS + 1) * 4096u);
                    for (int s = 0; s < JS; ++s) tma_load_2d(xs + st * SF + s * 1024, &tmX, 32 * s, r0, &full[st]);
                    tma_load_2d(xs + st * SF + JS * 1024, &tmU, 0, r0, &full[st]);
                }
            }
            __syncwarp();
        }
        return;
    }
    const int NSW = kCW / RG;  // strip slots per row group
    const int s = w % NSW, rg = w / NSW;
    const bool act = s < JS;
    const int pg = qperm(g);
    double acc[4][2][2];
#pragma unroll
    for (int e = 0; e < 4; ++e)
#pragma unroll
        for (int f = 0; f < 2; ++f) acc[e][f][0] = acc[e][f][1] = 0.0;
    unsigned vm = 0;
    for (int64_t i = 0, k = -1; i < mine; ++i) {
        if ((i & 31) == 0) vm = visit_mask(tflag, tgen, i, mine);
        if (!((vm >> (i & 31)) & 1u)) continue;
        ++k;
        const int st = (int)(k % kStages32);
        mbar_wait(&full[st], (uint32_t)((k / kStages32) & 1));
        const float *xt = xs + st * SF;
        const double *ut = reinterpret_cast<const double *>(xt + JS * 1024);
        if (act) {
            for (int kk = rg; kk < kTR / 4; kk += RG) {
                const int row = 4 * kk + t;
                const double2 b = *reinterpret_cast<const double2 *>(ut + swz(row, pg));         // US[row][2pg..]
                const float4 a = *reinterpret_cast<const float4 *>(xt + s * 1024 + swzf(row, pg));  // X[row][4pg..]
                const double av[4] = {(double)a.x, (double)a.y, (double)a.z, (double)a.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    dmma884(acc[e][0], av[e], b.x);
                    dmma884(acc[e][1], av[e], b.y);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
    }
    if (!act) return;
    double *slot = F_slots + ((int64_t)blockIdx.x * RG + rg) * J * R;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const int j = 32 * s + 4 * pg + e;
#pragma unroll
        for (int f = 0; f < 2; ++f)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const int r = 2 * qperm(2 * t + v) + f;
                if (j < J && r < R) slot[j * R + r] = acc[e][f][v];
            }
    }
}
