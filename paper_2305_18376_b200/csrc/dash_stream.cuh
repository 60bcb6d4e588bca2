// Streaming tall-skinny GEMMs over the update batch X (N x J, FP64), the two
// data-sized contractions of one DASH pass:
//
//   k_xv2     XV = X V              (stream.py:314-315)
//   k_fgemm2  F_cta = X^T US        (stream.py:321, US = U o w_slice(row))
//
// Both are persistent (one CTA per SM), warp-specialised: warp 8 is a TMA
// producer that streams X (one cp.async.bulk per row into a padded row pitch,
// so the DMMA fragment reads are conflict-free) and US (one bulk copy per
// tile) through a kStages-deep shared-memory ring; the 8 compute warps
// consume stages on "full" mbarriers and release them on "empty" mbarriers,
// multiplying on the FP64 tensor cores (mma.sync m8n8k4 f64 -> DMMA.8x8x4).
// V (J x R) stays resident in shared memory for the whole kernel; the F
// accumulators stay in registers and are written once per CTA (fixed-order
// slot reduction afterwards -> deterministic).
#pragma once

// (included inside dash_update.cu's anonymous namespace)

constexpr int kTR = 32;      // rows per tile
constexpr int kStages = 4;   // ring depth

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// mbar_wait with a suspend-time hint: a waiting warp sleeps in the barrier
// instead of re-issuing try_wait (long hand-off waits in warp-specialised
// kernels otherwise burn issue slots the working warps need).
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(20u)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void compute_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }  // 8 compute warps
constexpr int kCW = 8;  // compute warps; warp kCW is the producer
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// Issue the row copies of one tile: warp 0, lane l copies row l (and the matching
// US row when us != nullptr).  Lane 0 arms the barrier with the total byte count first.
__device__ __forceinline__ void issue_tile(const double *X, int64_t ldx, int64_t N, int J, const double *US, int R,
                                           int64_t tile, double *xs, int XP, double *uss, int UP, uint64_t *bar) {
    const int lane = lane_id();
    const int64_t r0 = tile * kTR;
    const int nr = (int)min((int64_t)kTR, N - r0);
    const uint32_t bytes = (uint32_t)nr * J * 8u + (US ? (uint32_t)nr * R * 8u : 0u);
    if (lane == 0) mbar_arrive_expect_tx(bar, bytes);
    __syncwarp();
    if (lane < nr) bulk_g2s(xs + lane * XP, X + (r0 + lane) * ldx, (uint32_t)J * 8u, bar);
    if (US && lane == 0) bulk_g2s(uss, US + r0 * R, (uint32_t)nr * R * 8u, bar);  // dense rows, pitch R
}

// producer warp: fill stage (i % kStages) once the compute warps released it
template <typename IssueFn>
__device__ __forceinline__ void produce(int64_t mine, uint64_t *full, uint64_t *empty, IssueFn issue) {
    for (int64_t i = 0; i < mine; ++i) {
        const int st = (int)(i % kStages);
        if (i >= kStages) mbar_wait(&empty[st], (uint32_t)(((i / kStages) - 1) & 1));
        fence_proxy_async();
        issue(i, st);
    }
}

template <int RP>
struct StreamSmem {
    static constexpr int UP = (RP % 16 == 0) ? RP + 8 : RP;  // US / V row pitch (conflict-free B frags)
    static __host__ __device__ int xp(int J) { return ((J + 7) / 8) * 8 + 4; }
    static __host__ __device__ size_t xv_bytes(int J) {
        return sizeof(double) * ((size_t)kStages * kTR * xp(J) + (size_t)((J + 7) / 8) * 8 * UP) + 16 * kStages + 64;
    }
    static __host__ __device__ size_t f_bytes(int J) {
        return sizeof(double) * ((size_t)kStages * kTR * xp(J) + (size_t)kStages * kTR * UP) + 16 * kStages + 64;
    }
};

// XV = X V.  8 warps: warp w -> 8-row block (w % 4) of the 32-row tile and
// half (w / 4) of the RP/8 column blocks (RP = 8: warps 4-7 split K instead).
template <int RP>
__global__ void __launch_bounds__(kCW * 32 + 32, 1) k_xv2(const double *__restrict__ X, int64_t ldx, int64_t N, int J,
                                                          const double *__restrict__ V, int R, double *__restrict__ XV) {
    using S = StreamSmem<RP>;
    constexpr int UP = S::UP, NB = RP / 8;
    extern __shared__ __align__(16) double sm[];
    const int XP = S::xp(J), JP = ((J + 7) / 8) * 8;
    double *xs = sm;                                  // kStages x kTR x XP
    double *vs = xs + (size_t)kStages * kTR * XP;     // JP x UP
    uint64_t *full = reinterpret_cast<uint64_t *>(vs + (size_t)JP * UP);
    uint64_t *empty = full + kStages;
    const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
    const int g = lane >> 2, t = lane & 3;
    for (int i = tid; i < kStages * kTR * (XP - J); i += blockDim.x) {
        const int row = i / (XP - J), c = J + i % (XP - J);
        xs[(size_t)row * XP + c] = 0.0;
    }
    for (int i = tid; i < JP * UP; i += blockDim.x) {
        const int j = i / UP, c = i % UP;
        vs[i] = (j < J && c < R) ? V[j * R + c] : 0.0;
    }
    if (tid == 0) {
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
        produce(mine, full, empty, [&](int64_t i, int st) {
            issue_tile(X, ldx, N, J, nullptr, R, blockIdx.x + i * gridDim.x, xs + (size_t)st * kTR * XP, XP, nullptr,
                       0, &full[st]);
        });
        return;
    }
    const int mb = w & 3, half = w >> 2;
    for (int64_t i = 0; i < mine; ++i) {
        const int st = (int)(i % kStages);
        mbar_wait(&full[st], (uint32_t)((i / kStages) & 1));
        const double *xt = xs + (size_t)st * kTR * XP;
        const int64_t r0 = (blockIdx.x + i * gridDim.x) * kTR;
        if constexpr (NB >= 2) {
            constexpr int NH = NB / 2;
            double acc[NH][2], acc2[NH][2];
#pragma unroll
            for (int n = 0; n < NH; ++n) acc[n][0] = acc[n][1] = acc2[n][0] = acc2[n][1] = 0.0;
            const double *arow = xt + (8 * mb + g) * XP + t;
            int kk = 0;
            for (; kk + 1 < JP / 4; kk += 2) {  // two independent accumulation chains
                const double a0 = arow[4 * kk], a1 = arow[4 * kk + 4];
#pragma unroll
                for (int n = 0; n < NH; ++n) {
                    dmma884(acc[n], a0, vs[(4 * kk + t) * UP + 8 * (half * NH + n) + g]);
                    dmma884(acc2[n], a1, vs[(4 * kk + 4 + t) * UP + 8 * (half * NH + n) + g]);
                }
            }
            if (kk < JP / 4) {
                const double a0 = arow[4 * kk];
#pragma unroll
                for (int n = 0; n < NH; ++n) dmma884(acc[n], a0, vs[(4 * kk + t) * UP + 8 * (half * NH + n) + g]);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
            const int64_t row = r0 + 8 * mb + g;
            if (row < N) {
#pragma unroll
                for (int n = 0; n < NH; ++n)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int col = 8 * (half * NH + n) + 2 * t + e;
                        if (col < R) XV[row * R + col] = acc[n][e] + acc2[n][e];
                    }
            }
        } else {
            // RP == 8: warps w and w+4 split K, then combine through shared memory
            double acc[2] = {0.0, 0.0};
            const double *arow = xt + (8 * mb + g) * XP + t;
            const int k4 = JP / 4, kh = (k4 + 1) / 2;
            for (int kk = half * kh; kk < min(k4, (half + 1) * kh); ++kk)
                dmma884(acc, arow[4 * kk], vs[(4 * kk + t) * UP + g]);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
            __shared__ double part[4][32][2];
            if (half == 1) {
                part[mb][lane][0] = acc[0];
                part[mb][lane][1] = acc[1];
            }
            compute_bar();
            if (half == 0) {
                const int64_t row = r0 + 8 * mb + g;
                if (row < N)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int col = 2 * t + e;
                        if (col < R) XV[row * R + col] = acc[e] + part[mb][lane][e];
                    }
            }
            compute_bar();
        }
    }
}

// F_cta = sum over this CTA's tiles of X^T US.  Accumulator tiles (JP/8 x RP/8)
// are dealt round-robin to the 8 warps (<= 8 per warp); written to slot blockIdx.x.
template <int RP, int MAXT>
__global__ void __launch_bounds__(kCW * 32 + 32, 1) k_fgemm2(const double *__restrict__ X, int64_t ldx, int64_t N,
                                                             int J, const double *__restrict__ US, int R,
                                                             double *__restrict__ F_slots) {
    using S = StreamSmem<RP>;
    constexpr int NB = RP / 8;
    extern __shared__ __align__(16) double sm[];
    const int XP = S::xp(J), JP = ((J + 7) / 8) * 8;
    const int UPd = R;  // US stage rows are dense (one bulk copy per tile)
    double *xs = sm;
    double *us = xs + (size_t)kStages * kTR * XP;     // kStages x kTR x S::UP (dense pitch R used)
    uint64_t *full = reinterpret_cast<uint64_t *>(us + (size_t)kStages * kTR * S::UP);
    uint64_t *empty = full + kStages;
    const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
    const int g = lane >> 2, t = lane & 3;
    for (int i = tid; i < kStages * kTR * (XP - J); i += blockDim.x) {
        const int row = i / (XP - J), c = J + i % (XP - J);
        xs[(size_t)row * XP + c] = 0.0;
    }
    if (tid == 0) {
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
        produce(mine, full, empty, [&](int64_t i, int st) {
            issue_tile(X, ldx, N, J, US, R, blockIdx.x + i * gridDim.x, xs + (size_t)st * kTR * XP, XP,
                       us + (size_t)st * kTR * S::UP, 0, &full[st]);
        });
        return;
    }
    const int ntile_acc = (JP / 8) * NB;
    double acc[MAXT][2];
#pragma unroll
    for (int q = 0; q < MAXT; ++q) acc[q][0] = acc[q][1] = 0.0;
    for (int64_t i = 0; i < mine; ++i) {
        const int st = (int)(i % kStages);
        mbar_wait(&full[st], (uint32_t)((i / kStages) & 1));
        double *xt = xs + (size_t)st * kTR * XP;
        double *ut = us + (size_t)st * kTR * S::UP;
        const int64_t r0 = (blockIdx.x + i * gridDim.x) * kTR;
        const int nr = (int)min((int64_t)kTR, N - r0);
        if (nr < kTR) {  // tail tile: stale (possibly uninitialised) rows must not contribute
            for (int e = tid; e < (kTR - nr) * UPd; e += kCW * 32) ut[nr * UPd + e] = 0.0;
            for (int e = tid; e < (kTR - nr) * XP; e += kCW * 32) xt[nr * XP + e] = 0.0;
            compute_bar();
        }
#pragma unroll
        for (int q = 0; q < MAXT; ++q) {
            const int p = w + kCW * q;
            if (p < ntile_acc) {
                const int mb = p / NB, nb = p % NB;
                const int col = 8 * nb + g;
#pragma unroll
                for (int kk = 0; kk < kTR / 4; ++kk) {
                    const double a = xt[(4 * kk + t) * XP + 8 * mb + g];
                    const double b = col < R ? ut[(4 * kk + t) * UPd + col] : 0.0;
                    dmma884(acc[q], a, b);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
    }
    double *slot = F_slots + (int64_t)blockIdx.x * J * R;
#pragma unroll
    for (int q = 0; q < MAXT; ++q) {
        const int p = w + kCW * q;
        if (p < ntile_acc) {
            const int mb = p / NB, nb = p % NB;
            const int j = 8 * mb + g;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int col = 8 * nb + 2 * t + e;
                if (j < J && col < R) slot[j * R + col] = acc[q][e];
            }
        }
    }
}
