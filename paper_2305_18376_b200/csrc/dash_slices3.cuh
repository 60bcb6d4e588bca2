// k_slices3: the per-slice phase (_kernels.py:62-144) for SMALL slices
// (<= kSmallRows rows), persistent and warp-autonomous.
//
// k_slices2 ran every CTA in lock-step rounds separated by __syncthreads, so
// each round's global-load latencies (metadata, W, D, XV) were exposed while
// the FP64 pipe idled.  Here every warp owns a static stream of units (one
// slice per RB-lane group, 32/RB slices per unit) and never waits for another
// warp: it loads the unit's metadata, issues cp.async copies of the slices'
// D columns and XV rows into its own shared staging, and runs the A-system
// sweep while those copies are in flight.  CTA barriers appear only in the
// prologue (vtv) and epilogue (per-CTA G slot, summed in fixed group order ->
// deterministic).  Same sweep / LU-fallback / SolveError chain as k_slices2.
// (included inside dash_update.cu's anonymous namespace)
#pragma once

#ifndef DASH_S3_CTAS
#define DASH_S3_CTAS 4
#endif
constexpr int kS3CtasPerSM = DASH_S3_CTAS;  // resident CTAs per SM (register budget 65536 / (128 x this))
constexpr double kS3Neumann = 1e-4;         // Neumann fast path bound on ||P d||: truncation O(rho^3) <= 1e-12
constexpr double kS3Neumann1 = 1e-6;        // below this the first-order term suffices: O(rho^2) <= 1e-12

// -sum_{z < n} a[z] x[z] in four interleaved chains combined in fixed order
template <int RB, typename X>
__device__ __forceinline__ double neg_dot4(const double (&a)[RB], const X &x, int n) {
    double q[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int z = 0; z < RB; ++z)
        if (z < n) q[z & 3] = fma(-a[z], x[z], q[z & 3]);
    return (q[0] + q[1]) + (q[2] + q[3]);
}

template <int RB>
struct S3 {
    static constexpr int NW = 4;
    static constexpr int GPW = 32 / RB;
    static constexpr int NG = NW * GPW;
    static constexpr int LDV = RB + 2;
    static constexpr int LDL = RB + 1;
    static constexpr int CAPW = 14;  // XV rows staged per group (longer slices read XV directly)
    // per group: buf[RB+2] (gathers; gj_solve scratch) | dn[RB*LDL] | xs[CAPW*RB]
    // per warp : gacc[RB*LDL] | lu[RB*LDL] | piv[RB].  RB = 16 (two groups): group 0
    // accumulates G into gacc, group 1 into lu (no turn-taking); the rare LU
    // fallback first folds lu into gacc and re-zeroes it afterwards.  RB < 16:
    // the warp's groups add into gacc in turn.
    //            (LU fallback scratch, used by one group at a time)
    // Per-lane rows use the odd pitch LDL = RB+1 (lane r's row r hits distinct banks).
    // per CTA after the warps: P = vtv^{-1} (RB x RB, symmetric, read by column) | ||P||_inf | ok
    // ~55 KB for RB = 16: four CTAs (16 warps) per SM.
    static constexpr int per_group = (RB + 2) + RB * LDL + CAPW * RB;
    static constexpr int per_warp = GPW * per_group + 2 * RB * LDL + RB;
    static constexpr int shared = RB * LDV;
    static constexpr int pinv = RB * RB + 2;
    __host__ __device__ static constexpr size_t bytes() { return sizeof(double) * (shared + NW * per_warp + pinv); }
    static_assert(shared % 2 == 0 && per_group % 2 == 0 && per_warp % 2 == 0 && (RB * LDL) % 2 == 0,
                  "group scratch must stay 16-byte aligned");
};

// lu_fallback for the groups with `need`, one group of the warp at a time (the
// LU scratch is per warp).  Rare path.
template <int RB>
__device__ __forceinline__ bool lu_fallback_seq(double (&a)[RB], double *lu, int *piv, int r, int R, bool need) {
    constexpr int GPW = 32 / RB;
    const int gme = lane_id() / RB;
    bool ok = true;
#pragma unroll 1
    for (int gi = 0; gi < GPW; ++gi) {
        const bool ng = need && gme == gi;
        if (__any_sync(FULL_MASK, ng)) {
            const bool o = lu_fallback<RB>(a, lu, piv, r, R, ng);
            if (gme == gi) ok = o;
        }
    }
    return ok;
}

// ---- device-side slice plan (R <= 16), once per update --------------------
// Stable counting sort of the batch positions by bucket: small slices
// (n <= kSmallRows) longest first (bucket kSmallRows - n), then big slices by
// 64-row size class, largest first.  Output: meta[M] = (r0, n, wrow | fresh <<
// 31, m) in plan order and plan_counts = {nsmall, nbig}.  Deterministic: per
// chunk histograms, a sequential scan, and a warp-ordered scatter.  No host
// work and no host round trip: the slice kernels read the counts on device.
constexpr int kPlanChunk = 256;                   // batch positions per chunk (one warp scatters a chunk)
constexpr int kBigClasses = 128;                  // 64-row classes, (64, 8192+]
constexpr int kPlanBuckets = kSmallRows + 1 + kBigClasses;

__device__ __forceinline__ int plan_bucket(int64_t n) {
    if (n <= kSmallRows) return kSmallRows - (int)n;
    const int64_t q = (n - 1) / 64 + 1;  // n in (kSmallRows, 64] -> class 1
    const int c = q < kBigClasses ? (int)q : kBigClasses;  // 1..kBigClasses
    return kSmallRows + 1 + (kBigClasses - c);
}

// hist[b][c]: bucket-b count of chunk c (bucket-major; one CTA of kPlanChunk threads per chunk)
// tflag (optional): tflag[t] = tgen for every 32-row tile holding a row of a
// small slice -- the tiles the small-row GEMMs must visit when big slices take
// the fused path (dash_bigx.cuh).  tgen changes every update, so stale marks
// never match and the array is never cleared (zeroed once at allocation).
__global__ void __launch_bounds__(kPlanChunk) k_plan_count(const int64_t *__restrict__ row_ptr, int M,
                                                           int *__restrict__ hist, uint32_t *__restrict__ tflag,
                                                           uint32_t tgen) {
    pdl_trigger();
    __shared__ int h[kPlanBuckets];
    for (int i = threadIdx.x; i < kPlanBuckets; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const int m = blockIdx.x * kPlanChunk + threadIdx.x;
    if (m < M) {
        const int64_t r0 = row_ptr[m], n = row_ptr[m + 1] - r0;
        atomicAdd(&h[plan_bucket(n)], 1);
        if (tflag != nullptr && n > 0 && n <= kSmallRows)
            for (int64_t t = r0 / 32; t <= (r0 + n - 1) / 32; ++t) tflag[t] = tgen;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kPlanBuckets; i += blockDim.x) hist[(size_t)i * gridDim.x + blockIdx.x] = h[i];
}

// One CTA per bucket b: off[b][c] = bucket-b positions in chunks < c
// (coalesced block scan over the chunks, tiles of 256 with a carry) and
// tot[b] = all bucket-b positions.  The bucket bases are a scan of tot,
// taken by each scatter warp itself.
constexpr int kScanThreads = 256;
__global__ void __launch_bounds__(kScanThreads) k_plan_scan(const int *__restrict__ hist, int nch,
                                                            int *__restrict__ off, int *__restrict__ tot) {
    pdl_wait();
    pdl_trigger();
    __shared__ int wsum[kScanThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, wq = tid >> 5;
    const int *h = hist + (size_t)blockIdx.x * nch;
    int *o = off + (size_t)blockIdx.x * nch;
    int carry = 0;
    for (int c0 = 0; c0 < nch; c0 += kScanThreads) {
        const int c = c0 + tid;
        const int v = c < nch ? h[c] : 0;
        int inc = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int u = __shfl_up_sync(FULL_MASK, inc, d);
            if (lane >= d) inc += u;
        }
        if (lane == 31) wsum[wq] = inc;
        __syncthreads();
        int wbase = 0, all = 0;
#pragma unroll
        for (int k = 0; k < kScanThreads / 32; ++k) {
            const int x = wsum[k];
            if (k < wq) wbase += x;
            all += x;
        }
        if (c < nch) o[c] = carry + wbase + inc - v;
        carry += all;
        __syncthreads();
    }
    if (tid == 0) tot[blockIdx.x] = carry;
}

// exclusive scan of tot[0..kPlanBuckets) by one warp into base[] (shared)
__device__ __forceinline__ void plan_bases(const int *__restrict__ tot, int *base, int lane) {
    constexpr int PER = (kPlanBuckets + 31) / 32;
    int v[PER], s = 0;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int b = lane * PER + k;
        v[k] = b < kPlanBuckets ? tot[b] : 0;
        s += v[k];
    }
    int inc = s;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int u = __shfl_up_sync(FULL_MASK, inc, d);
        if (lane >= d) inc += u;
    }
    int run = inc - s;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int b = lane * PER + k;
        if (b < kPlanBuckets) base[b] = run;
        run += v[k];
    }
}

// one warp per chunk (4 chunks per CTA): the chunk's loads are issued up
// front, then 32 positions at a time are ranked in order -> stable
__global__ void __launch_bounds__(128) k_plan_scatter(const int64_t *__restrict__ row_ptr,
                                                      const int32_t *__restrict__ state_row,
                                                      const uint8_t *__restrict__ is_new, int M, int nch,
                                                      const int *__restrict__ off, const int *__restrict__ tot,
                                                      int4 *__restrict__ meta, int *__restrict__ counts) {
    constexpr int ROUNDS = kPlanChunk / 32;
    pdl_wait();
    pdl_trigger();
    __shared__ int run_s[4][kPlanBuckets];
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    const int chunk = blockIdx.x * 4 + wq;
    if (chunk >= nch) return;
    int *run = run_s[wq];
    plan_bases(tot, run, lane);
    __syncwarp();
    if (chunk == 0 && lane == 0) {  // {nsmall, nbig}
        const int nsmall = run[kSmallRows + 1];
        counts[0] = nsmall;
        counts[1] = run[kPlanBuckets - 1] + tot[kPlanBuckets - 1] - nsmall;
    }
    for (int b = lane; b < kPlanBuckets; b += 32) run[b] += off[(size_t)b * nch + chunk];
    const int c0 = chunk * kPlanChunk;
    int64_t r0[ROUNDS];
    int nn[ROUNDS], sr[ROUNDS];
#pragma unroll
    for (int k = 0; k < ROUNDS; ++k) {
        const int m = c0 + 32 * k + lane;
        r0[k] = 0;
        nn[k] = -1;
        sr[k] = 0;
        if (m < M) {
            r0[k] = row_ptr[m];
            nn[k] = (int)(row_ptr[m + 1] - r0[k]);
            sr[k] = (int)((unsigned)state_row[m] | (is_new[m] ? 0x80000000u : 0u));
        }
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < ROUNDS; ++k) {
        const bool v = nn[k] >= 0;
        const int b = v ? plan_bucket(nn[k]) : -1 - lane;  // invalid lanes: unique keys
        const unsigned peers = __match_any_sync(FULL_MASK, b);
        const int rank = __popc(peers & ((1u << lane) - 1u));
        const int pos = v ? run[b] + rank : 0;
        __syncwarp();
        if (v && rank == 0) run[b] += __popc(peers);
        __syncwarp();
        if (v) meta[pos] = make_int4((int)r0[k], nn[k], sr[k], c0 + 32 * k + lane);
    }
}

template <int RB>
__global__ void __launch_bounds__(S3<RB>::NW * 32, kS3CtasPerSM) k_slices3(SliceParams p, const int4 *__restrict__ meta,
                                                                 const int *__restrict__ plan_counts) {
    using S = S3<RB>;
    constexpr int LDV = S::LDV, GPW = S::GPW, CAPW = S::CAPW;
    extern __shared__ __align__(16) double sm[];
    double *vtv_s = sm;
    const int lane = lane_id(), w = warp_id();
    const int r = lane % RB;
    const int gl = lane / RB;  // group within the warp
    double *wbase = sm + S::shared + w * S::per_warp;
    double *buf = wbase + gl * S::per_group;
    double *dns = buf + RB + 2;
    double *xs = dns + RB * S::LDL;
    double *gacc = wbase + GPW * S::per_group;
    double *lu = gacc + RB * S::LDL;
    int *piv = reinterpret_cast<int *>(lu + RB * S::LDL);
    const int R = p.R;
    constexpr bool kSplitG = (GPW == 2);
    double *gmine = (kSplitG && gl == 1) ? lu : gacc;  // this group's G accumulator
    if (gl == 0 || kSplitG) {
#pragma unroll
        for (int z = 0; z < RB; ++z) gmine[r * S::LDL + z] = 0.0;
    }
    // before an LU fallback borrows lu: fold group 1's G into gacc (fixed order)
    auto lu_borrow = [&]() {
        if (kSplitG) {
            if (gl == 1) {
#pragma unroll
                for (int z = 0; z < RB; ++z) gacc[r * S::LDL + z] += lu[r * S::LDL + z];
            }
            __syncwarp();
        }
    };
    auto lu_return = [&]() {
        if (kSplitG) {
            __syncwarp();
            if (gl == 1) {
#pragma unroll
                for (int z = 0; z < RB; ++z) lu[r * S::LDL + z] = 0.0;
            }
            __syncwarp();
        }
    };
    pdl_wait();     // XV, vtv (XV kernel) and the plan must be complete
    pdl_trigger();  // only now: the big-slice kernel relies on the same inputs without waiting
    for (int i = threadIdx.x; i < RB * LDV; i += blockDim.x) {
        const int a = i / LDV, b = i % LDV;
        vtv_s[i] = (a < R && b < R) ? p.vtv[a * R + b] : 0.0;
    }
    __syncthreads();
    const double *vrow = vtv_s + r * LDV;
    // ---- P = vtv^{-1} once per CTA (warp 0; both groups compute, group 0 writes):
    // the A system of every slice is S (vtv + sh S^-2) S, solved below by a
    // Neumann series around P when the ridge term is small (see the unit loop)
    double *P_s = sm + S::shared + S::NW * S::per_warp;
    if (w == 0) {
        double a[RB];
        double mx = r < R ? vrow[r] : 0.0;
#pragma unroll
        for (int off = RB / 2; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL_MASK, mx, off));
        const double im = (mx > 0.0 && isfinite(mx)) ? 1.0 / mx : 1.0;
#pragma unroll
        for (int z = 0; z < RB; ++z) a[z] = (r < R) ? ((z < R) ? vrow[z] * im : 0.0) : ((z == r) ? 1.0 : 0.0);
        const bool ok = sweep_inverse_unit<RB>(a, buf, r);
        double rs = 0.0;
#pragma unroll
        for (int z = 0; z < RB; ++z) {
            a[z] = (r < R && z < R) ? -a[z] * im : 0.0;  // P[r][z]
            rs += fabs(a[z]);
        }
#pragma unroll
        for (int off = RB / 2; off > 0; off >>= 1) rs = fmax(rs, __shfl_xor_sync(FULL_MASK, rs, off));
        if (gl == 0) {
#pragma unroll
            for (int z = 0; z < RB; ++z) P_s[z * RB + r] = a[z];  // column-major = row-major (symmetric)
            if (r == 0) {
                P_s[RB * RB] = rs;
                P_s[RB * RB + 1] = (ok && isfinite(rs) && !p.sweep_only) ? 1.0 : 0.0;
            }
        }
    }
    __syncthreads();
    const double pnorm = P_s[RB * RB];
    const bool pok = P_s[RB * RB + 1] != 0.0;

    const int nsmall = plan_counts[0];
    const int nunits = (nsmall + GPW - 1) / GPW;
    const int nwarps = gridDim.x * S::NW;
    // software pipeline: the next unit's metadata and W / C values are loaded
    // while the current unit computes, so a unit starts with one dependent
    // global round trip (the D / XV copies) instead of three.
    const int4 none = make_int4(0, 0, 0, 0);
    auto meta_of = [&](int unit) {
        const int j = unit * GPW + lane / RB;
        return (unit < nunits && j < nsmall) ? __ldg(meta + j) : none;
    };
    // raw (predicated) loads of the next unit's W / C entries: nothing consumes
    // them until that unit starts, so their latency hides behind this unit
    // (the bootstrap / dormant selects are applied at the consumer)
    auto sw_of = [&](const int4 &mt, bool act, double &sw, double &cw) {
        const int wr = mt.z & 0x7fffffff;
        const int64_t idx = (int64_t)wr * R + r;
        sw = 0.0;
        cw = 0.0;
        if (act && r < R) {
            sw = p.W[idx];
            cw = p.C[idx];
        }
    };
    int unit = blockIdx.x * S::NW + w;
    int4 nmeta = meta_of(unit);
    double nsw = 0.0, ncw = 0.0;
    sw_of(nmeta, unit < nunits && unit * GPW + lane / RB < nsmall, nsw, ncw);
    for (; unit < nunits; unit += nwarps) {
        const int j = unit * GPW + lane / RB;
        const bool active = j < nsmall;
        const int4 mt = nmeta;
        const int m = mt.w;
        const int64_t r0 = mt.x;
        const int64_t n = active ? mt.y : 0;
        const int wrow = mt.z & 0x7fffffff;
        const bool fresh = mt.z < 0;
        const bool real = active && r < R;
        const bool staged = n <= CAPW;
        const double s_r = real ? ((fresh && p.pass == 0) ? 1.0 : nsw) : 0.0;  // new slice: W bootstrap 1
        const double cold = (real && !fresh) ? ncw : 0.0;
        const int nxt = unit + nwarps;
        nmeta = meta_of(nxt);
        // ---- async prefetch: D column r (D symmetric; coalesced) and the XV rows
        if (real && !fresh) {
            const double *dcol = p.D + (int64_t)wrow * R * R + r;
            for (int z = 0; z < R; ++z) cp_async8(dns + r * S::LDL + z, dcol + (int64_t)z * R);
        }
        if (real && staged)
            for (int i = 0; i < (int)n; ++i) cp_async8(xs + i * RB + r, p.XV + (r0 + i) * R + r);

        // ---- A = vtv o s s^T + shift I  (_kernels.py:86-97)
        double s_all[RB];
        group_gather<RB>(s_r, buf, r, s_all);
        double sh;
        {
            double q4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int z = 0; z < RB; ++z)  // compile-time bound: s_all stays in registers
                if (z < R) q4[z & 3] = fma(vtv_s[z * LDV + z] * s_all[z], s_all[z], q4[z & 3]);
            sh = p.eps * ((q4[0] + q4[1]) + (q4[2] + q4[3])) / R;
        }
        // Fast path: A = S M S with M = vtv + diag(d), d_r = sh / s_r^2, so
        // u = A^{-1} (s o xv) = S^{-1} M^{-1} xv and M^{-1} = P - P d P + P d P d P - ...
        // Taken (warp-uniform) when rho = max_r d_r * ||P||_inf <= kS3Neumann
        // for every active slice of the warp: the dropped terms are O(rho^3)
        // relative (<= 1e-12).  Otherwise the exact sweep below.
        double a[RB];
        double im;       // sweep: 1 / max diag(A); fast path: 1 / s_r
        double dl = 0.0; // fast path: d_r
        bool fast, fast2;  // fast2: the second-order term is needed (rho > kS3Neumann1)
        {
            double q = 0.0, isr = 0.0;
            bool bad = false;
            if (real) {
                isr = rcp_nr(s_r);
                q = isr * isr;
                bad = !(s_r != 0.0) || !isfinite(q);
            }
            double qm = bad ? INFINITY : q;
#pragma unroll
            for (int off = RB / 2; off > 0; off >>= 1) qm = fmax(qm, __shfl_xor_sync(FULL_MASK, qm, off));
            const double rho = sh * qm * pnorm;
            const bool fg = !active || (pok && rho <= kS3Neumann);  // rho NaN / inf -> sweep
            fast = __all_sync(FULL_MASK, fg);
            fast2 = __any_sync(FULL_MASK, active && !(rho <= kS3Neumann1));
            im = isr;
            dl = real ? sh * q : 0.0;
        }
        if (fast) {
#pragma unroll
            for (int z = 0; z < RB; ++z) a[z] = -P_s[z * RB + r];  // -P[r][z]
            sw_of(nmeta, nxt < nunits && nxt * GPW + lane / RB < nsmall, nsw, ncw);  // next unit's s, c_old
        } else {
            // a <- -A^{-1} diag(s) by the sweep (LU fallback)
            {
                const double dg = real ? sh : 1.0;
                double mx = vrow[r] * s_r * s_r + dg;  // this lane's diagonal (padded lanes: 1)
#pragma unroll
                for (int off = RB / 2; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL_MASK, mx, off));
                im = (mx > 0.0 && isfinite(mx)) ? 1.0 / mx : 1.0;
                const double sr_im = s_r * im, dg_im = dg * im;
#pragma unroll
                for (int z = 0; z < RB; ++z) a[z] = vrow[z] * sr_im * s_all[z] + ((z == r) ? dg_im : 0.0);
            }
            const bool okA = sweep_inverse_unit<RB>(a, buf, r);
            if (!okA) im = 1.0;  // LU fallback below solves the unscaled A
            if (__any_sync(FULL_MASK, !okA)) {
                const double dg = real ? sh : 1.0;
#pragma unroll
                for (int z = 0; z < RB; ++z)
                    if (!okA) a[z] = vrow[z] * s_r * s_all[z] + ((z == r) ? dg : 0.0);
                if (!okA && r == 0) atomicAdd(p.fallbacks, 1u);
                lu_borrow();
                const bool okLU = lu_fallback_seq<RB>(a, lu, piv, r, R, !okA);
                lu_return();
                if (!okA && r == 0 && !okLU) report_error(p.err, m, DASH_E_SINGULAR);
            }
            sw_of(nmeta, nxt < nunits && nxt * GPW + lane / RB < nsmall, nsw, ncw);  // next unit's s, c_old
            group_gather<RB>(s_r, buf, r, s_all);
#pragma unroll
            for (int z = 0; z < RB; ++z) a[z] *= s_all[z];
        }
        cp_async_wait();
        __syncwarp();

        // ---- rows (_kernels.py:98-115): u, U, c, gram; u stashed over its xs row
        double c = 0.0, gram[RB];
#pragma unroll
        for (int z = 0; z < RB; ++z) gram[z] = 0.0;
        int64_t nmax = n;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1)
            nmax = max(nmax, (int64_t)__shfl_xor_sync(FULL_MASK, (long long)nmax, off));
        for (int64_t i = 0; i < nmax; ++i) {
            const bool valid = i < n;
            double u = 0.0, xrr = 0.0;
            if (valid) {  // y_r = -sum_z a[z] xv_z in 4 independent chains (DFMA latency, not a 16-deep chain)
                if (staged) {
                    const double *xr = xs + i * RB;
                    u = neg_dot4<RB>(a, xr, R);
                    xrr = r < R ? xr[r] : 0.0;
                } else {
                    const double *__restrict__ xr = p.XV + (r0 + i) * R;
                    u = neg_dot4<RB>(a, xr, R);
                    xrr = r < R ? __ldg(xr + r) : 0.0;
                }
            }
            if (fast) {  // u = S^{-1} (y - P d y + P d P d y), y = P xv (warp-uniform branch)
                double t[RB];
                group_gather<RB>(valid ? dl * u : 0.0, buf, r, t);
                const double c1 = neg_dot4<RB>(a, t, RB);  // (P d y)_r
                double c2 = 0.0;
                if (fast2) {
                    group_gather<RB>(valid ? dl * c1 : 0.0, buf, r, t);
                    c2 = neg_dot4<RB>(a, t, RB);  // (P d P d y)_r
                }
                u = (u - c1) + c2;
            }
            u *= im;
            if (!(valid && r < R)) u = 0.0;
            if (valid && r < R) {
                p.U[(r0 + i) * R + r] = u;
                c = fma(xrr, u, c);
            }
            double ua[RB];
            group_gather<RB>(u, buf, r, ua);
#pragma unroll
            for (int z = 0; z < RB; ++z) gram[z] = fma(u, ua[z], gram[z]);
            if (valid && staged) xs[i * RB + r] = u;  // all lanes read row i before the gather's sync
        }

        // ---- c, D accumulation and the S-row system (_kernels.py:103-135)
        const double cn = real ? p.lam * cold + c : 0.0;
        double *dn = dns + r * S::LDL;
        double drr = 0.0;
#pragma unroll
        for (int z = 0; z < RB; ++z) {
            double v = 0.0;
            if (real && z < R) v = p.lam * (fresh ? 0.0 : dn[z]) + gram[z];
            dn[z] = v;
            if (z == r) drr = v;
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
        {
            const double dg2 = real ? sh2 : 1.0;
#pragma unroll
            for (int z = 0; z < RB; ++z) a[z] = vrow[z] * dn[z] + ((z == r) ? dg2 : 0.0);
        }
        double wv;
        const bool okB = gj_solve<RB>(a, cn, buf, r, wv);  // w = B^{-1} c (buf: RB+2 scratch)
        if (!real) wv = 0.0;
        bool gok = okB && isfinite(wv);
        {
            const unsigned bal = __ballot_sync(FULL_MASK, !gok);
            const unsigned gmask = (RB == 32) ? FULL_MASK : (((1u << RB) - 1u) << ((lane / RB) * RB));
            gok = (bal & gmask) == 0;
        }
        if (__any_sync(FULL_MASK, !gok && active)) {
            const bool need = !gok && active;
            const double dg2 = real ? sh2 : 1.0;
#pragma unroll
            for (int z = 0; z < RB; ++z)
                if (need) a[z] = vrow[z] * dn[z] + ((z == r) ? dg2 : 0.0);
            if (need && r == 0) atomicAdd(p.fallbacks, 1u);
            lu_borrow();
            const bool okLU = lu_fallback_seq<RB>(a, lu, piv, r, R, need);
            lu_return();
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
                    if (z < R) p.D[(int64_t)wrow * R * R + (int64_t)z * R + r] = dn[z];  // column r
            }
            if (p.US != nullptr)
                for (int64_t i = 0; i < n; ++i)
                    p.US[(r0 + i) * R + r] = (staged ? xs[i * RB + r] : p.U[(r0 + i) * R + r]) * wv;
        }
        double wa[RB];
        group_gather<RB>(wv, buf, r, wa);
        if (kSplitG) {  // each group its own accumulator (lane r owns row r of it)
            if (active) {
#pragma unroll
                for (int z = 0; z < RB; ++z) gmine[r * S::LDL + z] = fma(gram[z] * wv, wa[z], gmine[r * S::LDL + z]);
            }
        } else {
#pragma unroll
            for (int gi = 0; gi < GPW; ++gi) {  // the warp's groups add into gacc in turn (fixed order)
                if (active && gl == gi) {
#pragma unroll
                    for (int z = 0; z < RB; ++z) gacc[r * S::LDL + z] = fma(gram[z] * wv, wa[z], gacc[r * S::LDL + z]);
                }
                __syncwarp();
            }
        }
    }
    // ---- per-CTA G slot, groups in order
    __syncthreads();
    double *slot = p.G_slots + (int64_t)blockIdx.x * R * R;
    for (int i = threadIdx.x; i < R * R; i += blockDim.x) {
        const int a = i / R, b = i % R;
        double acc = 0.0;
        for (int w2 = 0; w2 < S::NW; ++w2) {
            const double *g0 = sm + S::shared + w2 * S::per_warp + GPW * S::per_group;
            acc += g0[a * S::LDL + b];
            if (kSplitG) acc += g0[RB * S::LDL + a * S::LDL + b];  // the warp's lu region (group 1)
        }
        slot[i] = acc;
    }
}

template <int RB>
int launch_slices3(cudaStream_t st, int grid, const SliceParams &sp, const int4 *meta, const int *plan_counts) {
    const size_t smem = S3<RB>::bytes();
    ensure_smem_attr(k_slices3<RB>, smem);
    static const bool sweep_only = getenv("DASH_S3_SWEEP") != nullptr;  // A/B: exact sweep for every slice
    SliceParams q = sp;
    q.sweep_only = sweep_only ? 1 : 0;
    return launch_k(pdl_site("sl3"), k_slices3<RB>, grid, S3<RB>::NW * 32, smem, st, q, meta, plan_counts);
}
