// k_slices2: the per-slice phase of one DASH update (_kernels.py:62-144),
// designed for latency hiding:
//
//  * one slice per GROUP of RB lanes (RB = rank bucket 4/8/16/32), lane r of a
//    group owns index r of every per-slice vector and row r of every R x R
//    matrix -> 32/RB slices per warp in flight, 4 warps per CTA, several CTAs
//    per SM;
//  * both R x R ridge systems are inverted in place with the symmetric SWEEP
//    operator (Goodnight), one pivot per step: the pivot column is gathered
//    through 8 bytes of shared memory per lane, so a step is 1 STS + RB/2
//    LDS.128 + RB FMAs -- no serial triangular solves.  sweep(A) over all
//    pivots = -A^{-1};  U rows are then u_i = -(A^{-1} diag(s)) xv_i, one dot
//    product per lane, and w = -B^{-1} c.  SPD pivots are the same as
//    Cholesky's; a non-positive / non-finite pivot (or non-finite w) takes the
//    reference's fallback: LU with partial pivoting (numpy solve), then
//    SolveError on a zero pivot (stream.py:319-339, linalg.py:25-45);
//  * control flow is warp-uniform (row loops run to the warp's max row count
//    with per-group predicates), so plain __syncwarp() is safe.
//
// Items: {slice0, nslices, big, 0}.  Small items: each group takes slices
// g, g+NG, ... of the item.  Big item (one slice): every group inverts A
// (identical result), rows are interleaved over the groups, c / gram
// partials are reduced in group order, group 0 solves for w.
#pragma once

// (included inside dash_update.cu's anonymous namespace)

template <int RB>
struct S2 {
    static constexpr int NW = 4;             // warps per CTA
    static constexpr int GPW = 32 / RB;      // groups per warp
    static constexpr int NG = NW * GPW;      // groups per CTA
    static constexpr int LDV = RB + 2;       // vtv row pitch (16B aligned rows)
    static constexpr int LDL = RB + 1;       // LU scratch pitch
    static constexpr int CAPR = 128;         // XV rows staged per block
    static constexpr int CAPU = 16;          // u rows stashed per group (US write without re-reading U)
    // per group: buf[RB] | gacc[RB*LDL] | piv[RB] (as doubles) | dn[RB*LDL] | ust[CAPU*RB]
    // (per-lane rows at the odd pitch LDL: conflict-free; +pad keeps group bases 16B-aligned)
    static constexpr int per_group = RB + RB * LDL + RB + RB * LDL + CAPU * RB + ((RB * LDL * 2) & 1 ? 1 : 0);
    // union region (never live at the same time): staged XV rows [CAPR*RB] |
    // big-item partials red[NG*RB*(RB+1)] | per-group LU scratch [NG*RB*LDL]
    static constexpr int cmax(int a, int b) { return a > b ? a : b; }
    static constexpr int uni = cmax(CAPR * RB, cmax(NG * RB * (RB + 1), NG * RB * LDL));
    // shared: vtv[RB*LDV] | union | wsh[RB] (big item: w broadcast)
    static constexpr int shared = RB * LDV + uni + RB;
    __host__ __device__ static constexpr size_t bytes() { return sizeof(double) * (shared + NG * per_group); }
};

// all lanes of the group publish one value, every lane reads the RB-vector
template <int RB>
__device__ __forceinline__ void group_gather(double v, double *buf, int r, double (&out)[RB]) {
    buf[r] = v;
    __syncwarp();
    const double2 *b2 = reinterpret_cast<const double2 *>(buf);  // buf is 16-byte aligned
#pragma unroll
    for (int z = 0; z < RB / 2; ++z) {
        const double2 t = b2[z];
        out[2 * z] = t.x;
        out[2 * z + 1] = t.y;
    }
    __syncwarp();
}

// 8-byte async global->shared copy (no register staging); completes at cp_async_wait()
__device__ __forceinline__ void cp_async8(double *dst, const double *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src));
}
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_all;\n" ::); }

// In-place sweep of every pivot of the row-distributed symmetric matrix
// (lane r holds row r in a[]): a <- -A^{-1}.  Returns false on a
// non-positive or non-finite pivot.
template <int RB>
__device__ __forceinline__ bool sweep_inverse(double (&a)[RB], double *buf, int r) {
    bool ok = true;
#pragma unroll
    for (int k = 0; k < RB; ++k) {
        double col[RB];
        group_gather<RB>(a[k], buf, r, col);  // col[z] = A[z][k] = A[k][z]
        const double d = col[k];
        ok = ok && (d > 0.0) && isfinite(d);
        const double id = rcp_nr(d);
        const bool piv = (r == k);
        const double f = a[k] * id;
        // pivot row: a *= 1/d ; other rows: a -= (a_k/d) col   (one DMUL + one DFMA each)
        const double alpha = piv ? id : 1.0;
        const double beta = piv ? 0.0 : f;
#pragma unroll
        for (int z = 0; z < RB; ++z) {
            if (z == k) continue;
            a[z] = fma(-beta, col[z], a[z] * alpha);
        }
        a[k] = piv ? -id : f;
    }
    return ok;
}

// The same sweep for a matrix whose pivots are all <= 1 (the caller scales A
// by 1 / max diag: every pivot of an SPD matrix is at most its largest
// diagonal entry).  The pivot row's scaling a_k <- a_k / d is folded into the
// FMA every other row does, a <- a - f col, with f = 1 - 1/d on the pivot row
// (its row equals the gathered column: A stays symmetric), so each step costs
// RB DFMAs instead of RB DMULs + RB DFMAs.  With d <= 1, |1 - 1/d| <= 1/d and
// the folded form keeps full relative accuracy.  Returns a <- -(scaled A)^{-1}.
template <int RB>
__device__ __forceinline__ bool sweep_inverse_unit(double (&a)[RB], double *buf, int r) {
    bool ok = true;
#pragma unroll
    for (int k = 0; k < RB; ++k) {
        double col[RB];
        group_gather<RB>(a[k], buf, r, col);  // col[z] = A[z][k] = A[k][z]
        const double d = col[k];
        ok = ok && (d > 0.0) && isfinite(d);
        const double id = rcp_nr(d);
        const bool piv = (r == k);
        const double f = a[k] * id;
        const double beta = piv ? 1.0 - id : f;
#pragma unroll
        for (int z = 0; z < RB; ++z) {
            if (z == k) continue;
            a[z] = fma(-beta, col[z], a[z]);
        }
        a[k] = piv ? -id : f;
    }
    return ok;
}

// x = B^{-1} rhs for one right-hand side (lane r holds row r of the SPD B in
// a[] and rhs_r), by Gauss-Jordan elimination without normalising the pivot
// row: step k subtracts (a_i[k] / d_k) x (pivot row) from every other row,
// touching only the columns right of k; after RB steps the matrix is
// diag(d) and x_i = rhs_i / d_i.  The pivot row's trailing entries are read
// from the gathered column k (the trailing Schur complement is symmetric), so
// each step costs one shared store per lane and ~(RB-k)/2 LDS.128.  The
// pivot's reciprocal is computed one step ahead (off the critical path).
// Same success test as the sweep / Cholesky: every pivot > 0 and finite.
// pb: per-group scratch of >= RB + 2 doubles, 16-byte aligned.  a[] is
// destroyed.  ~136 DFMA per lane vs ~480 DP ops for the full sweep.
template <int RB>
__device__ __forceinline__ bool gj_solve(double (&a)[RB], double rhs, double *pb, int r, double &x) {
    bool ok = true;
    double idown = 0.0;
    double idn = rcp_nr(a[0]);  // lane 0's value is the first pivot's reciprocal
#pragma unroll
    for (int k = 0; k < RB; ++k) {
        const bool piv = (r == k);
        pb[r] = a[k];
        if (piv) *reinterpret_cast<double2 *>(pb + RB) = make_double2(rhs, idn);
        __syncwarp();
        const double2 ri = *reinterpret_cast<const double2 *>(pb + RB);  // (rhs_k, 1/d_k)
        const double2 *p2 = reinterpret_cast<const double2 *>(pb);
        double col[RB];
#pragma unroll
        for (int z = (k / 2) * 2; z < RB; z += 2) {
            const double2 v = p2[z / 2];
            col[z] = v.x;
            col[z + 1] = v.y;
        }
        const double d = col[k];
        ok = ok && (d > 0.0) && isfinite(d);
        if (piv) idown = ri.y;
        const double f = piv ? 0.0 : a[k] * ri.y;
#pragma unroll
        for (int z = k + 1; z < RB; ++z) a[z] = fma(-f, col[z], a[z]);
        rhs = fma(-f, ri.x, rhs);
        if (k + 1 < RB) idn = rcp_nr(a[k + 1]);
        __syncwarp();
    }
    x = rhs * idown;
    return ok;
}

// Fallback: -A^{-1} by LU with partial pivoting, for the groups with need
// set.  The caller stages the RB x RB matrix rows into lu (lane r -> row r,
// pitch LDL) and reads row r of the result back from lu afterwards; only
// shared-memory pointers cross the call, so no register array is ever
// materialised on the stack on the (common) path that never calls this.
template <int RB>
__device__ __noinline__ bool lu_neg_inverse_smem(double *lu, int *piv, int r, int R, bool need) {
    constexpr int LDL = RB + 1;
    __syncwarp();
    bool ok = true;
    if (need && r == 0) ok = lu_factor_serial(lu, LDL, R, piv);
    __syncwarp();
    double x[RB];  // column r of A^{-1} (= row r, symmetric); local memory, fallback path only
    for (int z = 0; z < RB; ++z) x[z] = (z == r) ? 1.0 : 0.0;
    if (need && r < R) lu_solve_serial(lu, LDL, R, piv, x);
    __syncwarp();
    if (need)
        for (int z = 0; z < RB; ++z) lu[r * LDL + z] = (r < R && z < R) ? -x[z] : (z == r ? -1.0 : 0.0);
    __syncwarp();
    return __shfl_sync(FULL_MASK, ok ? 1 : 0, (lane_id() / RB) * RB) != 0;
}

// stage a[] rows -> lu, invert (LU fallback), read back; warp-uniform call sites only
template <int RB>
__device__ __forceinline__ bool lu_fallback(double (&a)[RB], double *lu, int *piv, int r, int R, bool need) {
    constexpr int LDL = RB + 1;
    if (need) {
#pragma unroll
        for (int z = 0; z < RB; ++z) lu[r * LDL + z] = a[z];
    }
    const bool ok = lu_neg_inverse_smem<RB>(lu, piv, r, R, need);
    if (need) {
#pragma unroll
        for (int z = 0; z < RB; ++z) a[z] = lu[r * LDL + z];
    }
    return ok;
}

#ifdef DASH_DEBUG_TIMING
__device__ long long g_dbg[8192 * 8];
#define DBG_T(slot) do { if (threadIdx.x == 0 && blockIdx.x < 8192) g_dbg[blockIdx.x * 8 + (slot)] = clock64(); } while (0)
#else
#define DBG_T(slot) do {} while (0)
#endif

template <int RB>
__global__ void __launch_bounds__(S2<RB>::NW * 32, 3) k_slices2(SliceParams p) {
    DBG_T(0);
    using S = S2<RB>;
    constexpr int NG = S::NG, LDV = S::LDV;
    extern __shared__ double sm[];
    double *vtv_s = sm;
    double *red = vtv_s + RB * LDV;
    const int lane = lane_id(), w = warp_id();
    const int r = lane % RB;                 // index within the group
    const int gid = w * S::GPW + lane / RB;  // group id in the CTA
    double *gb = sm + S::shared + gid * S::per_group;
    double *buf = gb;
    double *gacc = buf + RB;
    int *piv = reinterpret_cast<int *>(gacc + RB * S::LDL);
    double *dns = gacc + RB * S::LDL + RB;  // d_new rows, lane r owns dns[r*LDL ..]
    double *ust = dns + RB * S::LDL;     // stashed u rows of a small slice
    double *xs = red;                   // staged XV rows (union)
    double *wsh = red + S::uni;         // big item: w broadcast to all groups
    double *lu = red + gid * RB * S::LDL;  // LU scratch (union; used only outside the row phase)
    const int R = p.R;
    for (int i = threadIdx.x; i < RB * LDV; i += blockDim.x) {
        const int a = i / LDV, b = i % LDV;
        vtv_s[i] = (a < R && b < R) ? p.vtv[a * R + b] : 0.0;
    }
#pragma unroll
    for (int z = 0; z < RB; ++z) gacc[r * S::LDL + z] = 0.0;
    __syncthreads();
    const double *vrow = vtv_s + r * LDV;  // row r of vtv (shared)

    const int4 item = p.items[blockIdx.x];
    const bool big = item.z != 0;
    const int nsl = item.y;
    const int rounds = big ? 1 : (nsl + NG - 1) / NG;
    DBG_T(1);

    for (int round = 0; round < rounds; ++round) {
        const int j = big ? 0 : round * NG + gid;
        const bool active = j < nsl;
        const int m = item.x + (active ? j : 0);
        const int64_t r0 = p.row_ptr[m];
        const int64_t n = active ? p.row_ptr[m + 1] - r0 : 0;
        const int wrow = p.state_row[m];
        const bool fresh = p.is_new[m] != 0;
        const bool real = active && r < R;

        // prefetch this slice's D row (cp.async -> dns) and c_old; consumed after the rows
        if (real && !fresh && (!big || gid == 0)) {
            // D is exactly symmetric: lane r reads COLUMN r (= row r), so the 16 lanes
            // of a group read 16 consecutive doubles per step (coalesced 128 B)
            const double *dcol = p.D + (int64_t)wrow * R * R + r;
            for (int z = 0; z < R; ++z) cp_async8(dns + r * S::LDL + z, dcol + (int64_t)z * R);
        }
        const double cold_pf = (real && !fresh) ? p.C[(int64_t)wrow * R + r] : 0.0;

        // ---- A = vtv o s s^T + shift I  (_kernels.py:86-96), then a <- -A^{-1} diag(s)
        const double s_r = real ? ((fresh && p.pass == 0) ? 1.0 : p.W[(int64_t)wrow * R + r]) : 0.0;
        double s_all[RB];
        group_gather<RB>(s_r, buf, r, s_all);
        double a[RB];
        {
            double sh = 0.0;
            _Pragma("unroll") for (int z = 0; z < RB; ++z)  // compile-time bound: s_all stays in registers
                if (z < R) sh += vtv_s[z * LDV + z] * s_all[z] * s_all[z];
            sh = p.eps * sh / R;
            const double dg = real ? sh : 1.0;  // padded / idle rows: identity
#pragma unroll
            for (int z = 0; z < RB; ++z) a[z] = vrow[z] * s_r * s_all[z] + ((z == r) ? dg : 0.0);
        }
        if (round == 0) DBG_T(2);
        bool okA = sweep_inverse<RB>(a, buf, r);
        if (round == 0) DBG_T(3);
        if (__any_sync(FULL_MASK, !okA)) {
            // rebuild A for the failing groups and invert by LU (reference: numpy solve)
            double sh = 0.0;
            _Pragma("unroll") for (int z = 0; z < RB; ++z)  // compile-time bound: s_all stays in registers
                if (z < R) sh += vtv_s[z * LDV + z] * s_all[z] * s_all[z];
            sh = p.eps * sh / R;
#pragma unroll
            for (int z = 0; z < RB; ++z) {
                double v = (r < R && z < R) ? vrow[z] * s_r * s_all[z] : (z == r ? 1.0 : 0.0);
                if (z == r && r < R) v += sh;
                if (!okA) a[z] = v;
            }
            if (!okA && r == 0) atomicAdd(p.fallbacks, 1u);
            const bool okLU = lu_fallback<RB>(a, lu, piv, r, R, !okA);
            if (!okA && r == 0 && !okLU) report_error(p.err, m, DASH_E_SINGULAR);
        }
        group_gather<RB>(s_r, buf, r, s_all);
#pragma unroll
        for (int z = 0; z < RB; ++z) a[z] *= s_all[z];  // a = -A^{-1} diag(s)

        // ---- rows: u_i = A^{-1}(s o xv_i); c and gram partials (_kernels.py:98-115)
        double c = 0.0, gram[RB];
#pragma unroll
        for (int z = 0; z < RB; ++z) gram[z] = 0.0;
        // rows of this round are contiguous in XV: stage them in blocks of CAPR
        // rows with coalesced loads, then every group reads its rows from smem
        const int64_t blk_lo = big ? r0 : p.row_ptr[item.x + round * NG];
        const int64_t blk_hi = big ? r0 + n : p.row_ptr[min(item.x + (round + 1) * NG, item.x + nsl)];
        for (int64_t base = blk_lo; base < blk_hi; base += S::CAPR) {
            const int64_t hi = min(blk_hi, base + (int64_t)S::CAPR);
            __syncthreads();
            {
                // rows staged with pitch RB (zero-padded when R < RB): 8 loads in flight per thread
                const double *src = p.XV + base * R;
                const int nrow = (int)(hi - base);
                constexpr int NT = S::NW * 32, UNR = 8;
                if (R == RB) {
                    const int tot = nrow * RB;
                    for (int e0 = threadIdx.x; e0 < tot; e0 += NT * UNR) {
                        double v[UNR];
#pragma unroll
                        for (int q = 0; q < UNR; ++q) {
                            const int e = e0 + q * NT;
                            v[q] = e < tot ? __ldg(src + e) : 0.0;
                        }
#pragma unroll
                        for (int q = 0; q < UNR; ++q) {
                            const int e = e0 + q * NT;
                            if (e < tot) xs[e] = v[q];
                        }
                    }
                } else {
                    const int tot = nrow * RB;
                    for (int e0 = threadIdx.x; e0 < tot; e0 += NT * UNR) {
                        double v[UNR];
#pragma unroll
                        for (int q = 0; q < UNR; ++q) {
                            const int e = e0 + q * NT;
                            const int rr = e / RB, z = e % RB;
                            v[q] = (e < tot && z < R) ? __ldg(src + rr * R + z) : 0.0;
                        }
#pragma unroll
                        for (int q = 0; q < UNR; ++q) {
                            const int e = e0 + q * NT;
                            if (e < tot) xs[e] = v[q];
                        }
                    }
                }
            }
            __syncthreads();
            int64_t lo_g, cnt;
            if (big) {
                lo_g = base + gid;
                cnt = (hi > lo_g) ? (hi - lo_g + NG - 1) / NG : 0;
            } else {
                lo_g = max(r0, base);
                cnt = max((int64_t)0, min(r0 + n, hi) - lo_g);
            }
            int64_t nmax = cnt;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1)
                nmax = max(nmax, (int64_t)__shfl_xor_sync(FULL_MASK, (long long)nmax, off));
            for (int64_t i = 0; i < nmax; ++i) {
                const bool valid = i < cnt;
                const int64_t row = big ? lo_g + i * NG : lo_g + i;
                const double2 *xr2 = reinterpret_cast<const double2 *>(xs + (valid ? (row - base) * RB : 0));
                double u = 0.0, xrr = 0.0;
#pragma unroll
                for (int z = 0; z < RB / 2; ++z) {
                    const double2 t = xr2[z];
                    u = fma(-a[2 * z], t.x, u);
                    u = fma(-a[2 * z + 1], t.y, u);
                    if (2 * z == r) xrr = t.x;
                    if (2 * z + 1 == r) xrr = t.y;
                }
                if (!(valid && r < R)) u = 0.0;
                if (valid && r < R) {
                    p.U[row * R + r] = u;
                    c = fma(xrr, u, c);
                }
                if (!big && valid && row - r0 < S::CAPU) ust[(row - r0) * RB + r] = u;
                double ua[RB];
                group_gather<RB>(u, buf, r, ua);
#pragma unroll
                for (int z = 0; z < RB; ++z) gram[z] = fma(u, ua[z], gram[z]);
            }
        }
        __syncthreads();

        if (round == 0) DBG_T(4);
        bool owner = true;
        if (big) {
            double *mine = red + gid * RB * (RB + 1) + r * (RB + 1);
#pragma unroll
            for (int z = 0; z < RB; ++z) mine[z] = gram[z];
            mine[RB] = c;
            __syncthreads();
            owner = (gid == 0);
            if (owner) {
                c = 0.0;
#pragma unroll
                for (int z = 0; z < RB; ++z) gram[z] = 0.0;
                for (int g2 = 0; g2 < NG; ++g2) {
                    const double *o = red + g2 * RB * (RB + 1) + r * (RB + 1);
#pragma unroll
                    for (int z = 0; z < RB; ++z) gram[z] += o[z];
                    c += o[RB];
                }
            }
        }
        // ---- c, D accumulation and the S-row system (_kernels.py:103-135)
        // (warp-uniform: for big items only group 0's lanes are `owner`, in warp 0)
        if (!big || w == 0) {
            const bool live = owner && active;
            const bool lreal = live && r < R;
            const double cold = (lreal && !fresh) ? cold_pf : 0.0;
            const double cn = lreal ? p.lam * cold + c : 0.0;
            cp_async_wait();
            __syncwarp();
            double *dn = dns + r * S::LDL;
            double drr = 0.0;
#pragma unroll
            for (int z = 0; z < RB; ++z) {
                double v = 0.0;
                if (lreal && z < R) {
                    const double dold = fresh ? 0.0 : dn[z];
                    v = p.lam * dold + gram[z];
                }
                dn[z] = v;
                if (z == r) drr = v;
            }
            // shift += vtv[r,r] * d_new[r,r] in the reference's order (_kernels.py:121-124)
            const double vrr = vrow[r];
            double sh2;
            {
                double vdd[RB];
                group_gather<RB>(lreal ? vrr * drr : 0.0, buf, r, vdd);
                double dsum = 0.0;
#pragma unroll
                for (int z = 0; z < RB; ++z)
                    if (z < R) dsum += vdd[z];
                sh2 = p.eps * dsum / R;
            }
            {
                const double dg2 = lreal ? sh2 : 1.0;
#pragma unroll
                for (int z = 0; z < RB; ++z) a[z] = vrow[z] * dn[z] + ((z == r) ? dg2 : 0.0);
            }
            if (round == 0) DBG_T(5);
            bool okB = sweep_inverse<RB>(a, buf, r);
            if (round == 0) DBG_T(6);
            double call[RB];
            group_gather<RB>(cn, buf, r, call);
            double wv = 0.0;
#pragma unroll
            for (int z = 0; z < RB; ++z) wv = fma(-a[z], call[z], wv);
            if (!lreal) wv = 0.0;
            bool fin = isfinite(wv);
            // group-wide verdict
            bool gok = okB && fin;
            {
                unsigned bal = __ballot_sync(FULL_MASK, !gok);
                const unsigned gmask = (RB == 32) ? FULL_MASK : (((1u << RB) - 1u) << ((lane / RB) * RB));
                gok = (bal & gmask) == 0;
            }
            if (__any_sync(FULL_MASK, !gok && live)) {
                const bool need = !gok && live;
#pragma unroll
                for (int z = 0; z < RB; ++z) {
                    double v = (lreal && z < R) ? vrow[z] * dn[z] : (z == r ? 1.0 : 0.0);
                    if (z == r && lreal) v += sh2;
                    if (need) a[z] = v;
                }
                if (need && r == 0) atomicAdd(p.fallbacks, 1u);
                const bool okLU = lu_fallback<RB>(a, lu, piv, r, R, need);
                if (need && r == 0 && !okLU) report_error(p.err, m, DASH_E_SINGULAR);
                double wv2 = 0.0;
#pragma unroll
                for (int z = 0; z < RB; ++z) wv2 = fma(-a[z], call[z], wv2);
                if (need) wv = lreal ? wv2 : 0.0;
                if (need && lreal && !isfinite(wv)) report_error(p.err, m, DASH_E_NONFINITE);
            }
            if (lreal) {
                p.W[(int64_t)wrow * R + r] = wv;
                if (p.final_pass) {
                    p.C[(int64_t)wrow * R + r] = cn;
#pragma unroll
                    for (int z = 0; z < RB; ++z)
                        if (z < R) p.D[(int64_t)wrow * R * R + (int64_t)z * R + r] = dn[z];  // column r (= row r)
                }
            }
            // ---- US = U o w for the F GEMM (small items: this group's own rows,
            // re-read from the U it wrote; big items: after the w broadcast below)
            if (p.US != nullptr && !big) {
                int64_t nm = live ? n : 0, nmx = nm;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1)
                    nmx = max(nmx, (int64_t)__shfl_xor_sync(FULL_MASK, (long long)nmx, off));
                for (int64_t i = 0; i < nmx; ++i)
                    if (i < nm && lreal)
                        p.US[(r0 + i) * R + r] = (i < S::CAPU ? ust[i * RB + r] : p.U[(r0 + i) * R + r]) * wv;
            }
            if (big && owner && r < RB) wsh[r] = lreal ? wv : 0.0;
            // ---- G contribution gram o w w^T (_kernels.py:139-143)
            double wa[RB];
            group_gather<RB>(wv, buf, r, wa);
            if (live) {
#pragma unroll
                for (int z = 0; z < RB; ++z) gacc[r * S::LDL + z] = fma(gram[z] * wv, wa[z], gacc[r * S::LDL + z]);
            }
        }
        if (big) {
            __syncthreads();
            if (p.US != nullptr) {
                const double wr = (r < R) ? wsh[r] : 0.0;
#pragma unroll 8
                for (int64_t row = r0 + gid; row < r0 + n; row += NG)
                    if (r < R) p.US[row * R + r] = p.U[row * R + r] * wr;
            }
        }
    }

    // ---- per-CTA G slot: groups summed in order
    __syncthreads();
    DBG_T(7);
    double *slot = p.G_slots + (int64_t)blockIdx.x * R * R;
    for (int i = threadIdx.x; i < R * R; i += blockDim.x) {
        const int a = i / R, b = i % R;
        double acc = 0.0;
        for (int g2 = 0; g2 < NG; ++g2) acc += sm[S::shared + g2 * S::per_group + RB + a * S::LDL + b];
        slot[i] = acc;
    }
}

template <int RB>
int launch_slices2(cudaStream_t st, int nitems, const SliceParams &sp) {
    const size_t smem = S2<RB>::bytes();
    ensure_smem_attr(k_slices2<RB>, smem);
    k_slices2<RB><<<nitems, S2<RB>::NW * 32, smem, st>>>(sp);
    return cudaGetLastError() == cudaSuccess ? 0 : DASH_E_CUDA;
}
