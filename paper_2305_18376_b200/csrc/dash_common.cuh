// Device building blocks shared by the DASH kernels (sm_100a, FP64).
//
//  * dmma884     -- FP64 tensor-core MMA (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4;
//                   tcgen05 has no f64 kind, DMMA is Blackwell's FP64 tensor path)
//  * warp solvers for the RB x RB ridge systems of one slice: Cholesky with
//                   the matrix held one row per lane (lane i = row i), factor
//                   kept in shared memory for many right-hand sides, and an LU
//                   (partial pivoting) fallback -- the reference's chain
//                   "numba Cholesky, on failure numpy/LAPACK LU, on singular
//                   SolveError" (_kernels.py:27-59, stream.py:319-339,
//                   linalg.py:25-45).
//
// Rank padding: a system of rank R <= RB is embedded as diag(A, I); the
// elimination never mixes the identity block into the real block, so the
// real R x R part of every result is exactly what an unpadded solve gives.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define FULL_MASK 0xffffffffu

namespace dash {

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
    asm volatile(
        "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c[0]), "+d"(c[1])
        : "d"(a), "d"(b));
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// 1/d to within 1 ulp: hardware reciprocal seed + two Newton steps (no IEEE
// division subroutine on a solver's critical path)
__device__ __forceinline__ double rcp_nr(double d) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    double e = fma(-d, r, 1.0);
    r = fma(r, e, r);
    e = fma(-d, r, 1.0);
    return fma(r, e, r);
}

// 1 / sqrt(d) to ~1 ulp for d > 0 (NaN / inf otherwise -- the caller's SPD test has
// already failed then): rsqrt.approx (2^-22) + two Newton steps y += y (1 - d y^2) / 2
__device__ __forceinline__ double rsqrt_nr(double d) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    double e = fma(-d * y, y, 1.0);
    y = fma(0.5 * y, e, y);
    e = fma(-d * y, y, 1.0);
    return fma(0.5 * y, e, y);
}

// Programmatic dependent launch (sm_90+): a kernel launched with the
// programmatic-serialization attribute may start while its predecessor in the
// stream is still running; pdl_wait() blocks until that predecessor has
// completed and its writes are visible, pdl_trigger() lets this kernel's own
// successor begin launching.  Every kernel on the PDL chain calls pdl_wait()
// in every CTA before it exits, so completion stays transitive.  Both are
// no-ops for a normally launched kernel.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }

__device__ __forceinline__ bool finite_d(double x) { return isfinite(x); }

// Error slot (one u64, ~0 = none): key = (position << 4) | code, so atomicMin
// keeps the first failing slice in batch order; the V solve (pos = -1) maps
// to kPosV, after every slice, as in the reference where the V solve runs last.
constexpr long long kPosV = 1ll << 40;
__device__ __forceinline__ void report_error(unsigned long long *err, long long pos, int code) {
    if (pos < 0) pos = kPosV;
    unsigned long long key = ((unsigned long long)pos << 4) | (unsigned long long)code;
    atomicMin(err, key);
}

// ---------------------------------------------------------------------------
// Cholesky of a register-resident RB x RB SPD matrix: lane i (< RB) holds row
// i in row[0..RB).  Right-looking; the update order a_ij -= l_ik l_jk for
// k = 0..j-1 is the reference's (_kernels.py:34-46).  On return row[] holds
// row i of L (upper part garbage) and L / 1/diag are also stored to shared
// memory.  Returns false (warp-uniform) if a pivot is not positive/finite.
// ---------------------------------------------------------------------------
template <int RB>
__device__ __forceinline__ bool chol_regs(double (&row)[RB], double *Lsm, int ld, double *dinv) {
    const int lane = lane_id();
    bool ok = true;
#pragma unroll
    for (int j = 0; j < RB; ++j) {
        double d = __shfl_sync(FULL_MASK, row[j], j);
        ok = ok && (d > 0.0) && finite_d(d);
        const double inv = rsqrt_nr(d);  // no IEEE sqrt / division on the column chain
        const double piv = d * inv;
        if (lane > j) row[j] = row[j] * inv;
        if (lane == j) row[j] = piv;
        if (lane == 0) dinv[j] = inv;
#pragma unroll
        for (int k = j + 1; k < RB; ++k) {
            double lkj = __shfl_sync(FULL_MASK, row[j], k);
            if (lane >= k) row[k] = fma(-row[j], lkj, row[k]);
        }
    }
    if (lane < RB) {
#pragma unroll
        for (int z = 0; z < RB; ++z) Lsm[lane * ld + z] = (z <= lane) ? row[z] : 0.0;
    }
    __syncwarp();
    return ok;
}

// Shared-memory load the compiler may not hoist out of loops (keeps the
// fully-unrolled triangular solves from caching all of L in registers).
__device__ __forceinline__ double lds_nohoist(const double *p) {
    double v;
    asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
    return v;
}

// Solve (L L^T) x = b for one right-hand side per lane (b in registers),
// L from shared memory (all lanes read the same element: broadcast).
template <int RB>
__device__ __forceinline__ void chol_solve_lane(const double *L, int ld, const double *dinv,
                                                double (&b)[RB]) {
#pragma unroll
    for (int k = 0; k < RB; ++k) {
        b[k] *= lds_nohoist(dinv + k);
#pragma unroll
        for (int i = k + 1; i < RB; ++i) b[i] = fma(-lds_nohoist(L + i * ld + k), b[k], b[i]);
    }
#pragma unroll
    for (int k = RB - 1; k >= 0; --k) {
        b[k] *= lds_nohoist(dinv + k);
#pragma unroll
        for (int i = 0; i < k; ++i) b[i] = fma(-lds_nohoist(L + k * ld + i), b[k], b[i]);
    }
}

// Single right-hand side distributed one entry per lane (lane i holds b_i):
// forward substitution uses the lane's own L row in registers, back
// substitution reads column entries L[k][lane] from shared memory.
template <int RB>
__device__ __forceinline__ double chol_solve_dist(const double (&row)[RB], const double *L, int ld,
                                                  const double *dinv, double b) {
    const int lane = lane_id();
#pragma unroll
    for (int k = 0; k < RB; ++k) {
        double yk = __shfl_sync(FULL_MASK, b, k) * dinv[k];
        if (lane == k) b = yk;
        if (lane > k) b = fma(-row[k], yk, b);
    }
#pragma unroll
    for (int k = RB - 1; k >= 0; --k) {
        double xk = __shfl_sync(FULL_MASK, b, k) * dinv[k];
        if (lane == k) b = xk;
        if (lane < k && lane < RB) b = fma(-L[k * ld + lane], xk, b);
    }
    return b;
}

// ---------------------------------------------------------------------------
// LU with partial pivoting, executed by lane 0 on a shared-memory matrix
// (rare fallback path).  A is n x n (ld), overwritten by L\U, piv[k] = row
// swapped into position k.  Returns false when a pivot is exactly zero
// (LAPACK getrf's "singular", which makes numpy raise LinAlgError).
// ---------------------------------------------------------------------------
__device__ inline bool lu_factor_serial(double *A, int ld, int n, int *piv) {
    bool ok = true;
    for (int k = 0; k < n; ++k) {
        int p = k;
        double best = fabs(A[k * ld + k]);
        for (int i = k + 1; i < n; ++i) {
            double v = fabs(A[i * ld + k]);
            if (v > best) { best = v; p = i; }
        }
        piv[k] = p;
        if (!(best > 0.0)) { ok = false; continue; }
        if (p != k)
            for (int j = 0; j < n; ++j) {
                double t = A[k * ld + j];
                A[k * ld + j] = A[p * ld + j];
                A[p * ld + j] = t;
            }
        double inv = 1.0 / A[k * ld + k];
        for (int i = k + 1; i < n; ++i) {
            double l = A[i * ld + k] * inv;
            A[i * ld + k] = l;
            for (int j = k + 1; j < n; ++j) A[i * ld + j] = fma(-l, A[k * ld + j], A[i * ld + j]);
        }
    }
    return ok;
}

// Solve with the LU factors for one right-hand side stored in x[0..n) (any
// memory space; used on per-lane shared scratch).
__device__ inline void lu_solve_serial(const double *A, int ld, int n, const int *piv, double *x) {
    for (int k = 0; k < n; ++k) {
        int p = piv[k];
        if (p != k) { double t = x[k]; x[k] = x[p]; x[p] = t; }
    }
    for (int i = 0; i < n; ++i) {
        double s = x[i];
        for (int k = 0; k < i; ++k) s = fma(-A[i * ld + k], x[k], s);
        x[i] = s;
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = x[i];
        for (int k = i + 1; k < n; ++k) s = fma(-A[i * ld + k], x[k], s);
        x[i] = s / A[i * ld + i];
    }
}

// Butterfly sum of a register vector across the warp (every lane ends with the total).
template <int RB>
__device__ __forceinline__ void warp_allreduce(double (&v)[RB]) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
        for (int r = 0; r < RB; ++r) v[r] += __shfl_xor_sync(FULL_MASK, v[r], off);
    }
}

}  // namespace dash
