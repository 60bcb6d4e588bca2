// k_slices_cta: the per-slice phase for large ranks (RB = 64), one CTA of 256
// threads per slice -- the R x R systems (R up to 64) live in shared memory and
// are inverted with the same symmetric sweep as k_slices2, every thread owning
// RB*RB/256 fixed matrix elements.  Same math / fallback chain as the reference
// (_kernels.py:62-144; LU + SolveError on failure, stream.py:319-339).
// (included inside dash_update.cu's anonymous namespace)
#pragma once

template <int RB>
struct SC {
    static constexpr int NT = 256;
    static constexpr int LDM = RB + 1;
    static constexpr int EPT = RB * RB / NT;  // matrix elements per thread
    static constexpr int CH = 32;             // rows per chunk
    // M[RB*LDM] | xc[CH*RB] | uc[CH*RB] | vec: s, c, w, dd, red[NT] | piv
    static constexpr int doubles = RB * LDM + 2 * CH * RB + 4 * RB + NT + RB;
    static constexpr size_t bytes() { return sizeof(double) * doubles; }
};

// -A^{-1} in place by sweeping every pivot; element ownership e = tid + NT*q.
template <int RB>
__device__ __forceinline__ bool cta_sweep(double *M) {
    using S = SC<RB>;
    constexpr int LDM = S::LDM;
    bool ok = true;
    for (int k = 0; k < RB; ++k) {
        __syncthreads();
        const double d = M[k * LDM + k];
        ok = ok && (d > 0.0) && isfinite(d);
        const double id = rcp_nr(d);
        double nv[S::EPT];
#pragma unroll
        for (int q = 0; q < S::EPT; ++q) {
            const int e = threadIdx.x + S::NT * q, i = e / RB, j = e % RB;
            const double mij = M[i * LDM + j];
            double v;
            if (i == k && j == k) v = -id;
            else if (i == k) v = mij * id;
            else if (j == k) v = mij * id;
            else v = fma(-M[i * LDM + k] * id, M[k * LDM + j], mij);
            nv[q] = v;
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < S::EPT; ++q) {
            const int e = threadIdx.x + S::NT * q;
            M[(e / RB) * LDM + (e % RB)] = nv[q];
        }
    }
    __syncthreads();
    return ok;
}

// fallback: M <- -A^{-1} via LU with partial pivoting (thread 0 factors; thread r
// solves column r).  Returns false on a zero pivot.
template <int RB>
__device__ bool cta_lu_neg_inverse(double *M, int *piv, int R, double *red) {
    using S = SC<RB>;
    __shared__ int okf;
    if (threadIdx.x == 0) okf = lu_factor_serial(M, S::LDM, R, piv) ? 1 : 0;
    __syncthreads();
    double x[RB];
    const int r = threadIdx.x;
    if (r < RB) {
        for (int z = 0; z < RB; ++z) x[z] = (z == r) ? 1.0 : 0.0;
        if (r < R) lu_solve_serial(M, S::LDM, R, piv, x);
    }
    __syncthreads();
    if (r < RB)
        for (int z = 0; z < RB; ++z) M[z * S::LDM + r] = (r < R && z < R) ? -x[z] : (z == r ? -1.0 : 0.0);
    __syncthreads();
    (void)red;
    return okf != 0;
}

template <int RB>
__global__ void __launch_bounds__(256, 2) k_slices_cta(SliceParams p) {
    using S = SC<RB>;
    constexpr int LDM = S::LDM, NT = S::NT, EPT = S::EPT, CH = S::CH;
    extern __shared__ double sm[];
    double *M = sm;
    double *xc = M + RB * LDM;
    double *uc = xc + CH * RB;
    double *sv = uc + CH * RB, *cv = sv + RB, *wv = cv + RB, *dd = wv + RB, *red = dd + RB;
    int *piv = reinterpret_cast<int *>(red + NT);
    const int tid = threadIdx.x, R = p.R;
    const int m = p.items[blockIdx.x].x;  // one slice per item
    const int64_t r0 = p.row_ptr[m], n = p.row_ptr[m + 1] - r0;
    const int wrow = p.state_row[m];
    const bool fresh = p.is_new[m] != 0;
    if (tid < RB) sv[tid] = tid < R ? ((fresh && p.pass == 0) ? 1.0 : p.W[(int64_t)wrow * R + tid]) : 0.0;
    __syncthreads();
    // ---- A = vtv o s s^T + shift I
    double sh = 0.0;
    for (int z = 0; z < R; ++z) sh += p.vtv[z * R + z] * sv[z] * sv[z];
    sh = p.eps * sh / R;
    for (int e = tid; e < RB * RB; e += NT) {
        const int i = e / RB, j = e % RB;
        double v = (i < R && j < R) ? p.vtv[i * R + j] * sv[i] * sv[j] : (i == j ? 1.0 : 0.0);
        if (i == j && i < R) v += sh;
        M[i * LDM + j] = v;
    }
    bool ok = cta_sweep<RB>(M);
    if (!__syncthreads_and(ok)) {
        if (tid == 0) atomicAdd(p.fallbacks, 1u);
        for (int e = tid; e < RB * RB; e += NT) {
            const int i = e / RB, j = e % RB;
            double v = (i < R && j < R) ? p.vtv[i * R + j] * sv[i] * sv[j] : (i == j ? 1.0 : 0.0);
            if (i == j && i < R) v += sh;
            M[i * LDM + j] = v;
        }
        __syncthreads();
        if (!cta_lu_neg_inverse<RB>(M, piv, R, red) && tid == 0) report_error(p.err, m, DASH_E_SINGULAR);
    }
    // M <- -A^{-1} diag(s)
    for (int e = tid; e < RB * RB; e += NT) M[(e / RB) * LDM + e % RB] *= sv[e % RB];
    __syncthreads();

    // ---- rows: u = A^{-1}(s o xv); c, gram (thread owns gram elements e = tid + NT q)
    double gram[EPT];
#pragma unroll
    for (int q = 0; q < EPT; ++q) gram[q] = 0.0;
    double c = 0.0;  // thread tid < RB owns c_tid
    for (int64_t c0 = 0; c0 < n; c0 += CH) {
        const int nr = (int)min((int64_t)CH, n - c0);
        for (int e = tid; e < CH * RB; e += NT) {
            const int i = e / RB, z = e % RB;
            xc[e] = (i < nr && z < R) ? p.XV[(r0 + c0 + i) * R + z] : 0.0;
        }
        __syncthreads();
        for (int e = tid; e < CH * RB; e += NT) {
            const int i = e / RB, r = e % RB;
            double u = 0.0;
            if (i < nr && r < R) {
                for (int z = 0; z < R; ++z) u = fma(-M[r * LDM + z], xc[i * RB + z], u);
                p.U[(r0 + c0 + i) * R + r] = u;
            }
            uc[e] = u;
        }
        __syncthreads();
        if (tid < R)
            for (int i = 0; i < nr; ++i) c = fma(xc[i * RB + tid], uc[i * RB + tid], c);
#pragma unroll
        for (int q = 0; q < EPT; ++q) {
            const int e = tid + NT * q, a = e / RB, b = e % RB;
            double acc = gram[q];
            for (int i = 0; i < nr; ++i) acc = fma(uc[i * RB + a], uc[i * RB + b], acc);
            gram[q] = acc;
        }
        __syncthreads();
    }
    // ---- c, D accumulation and the S-row system
    if (tid < RB) cv[tid] = tid < R ? p.lam * (fresh ? 0.0 : p.C[(int64_t)wrow * R + tid]) + c : 0.0;
    double dn[EPT];
#pragma unroll
    for (int q = 0; q < EPT; ++q) {
        const int e = tid + NT * q, a = e / RB, b = e % RB;
        double v = 0.0;
        if (a < R && b < R) v = p.lam * (fresh ? 0.0 : p.D[(int64_t)wrow * R * R + a * R + b]) + gram[q];
        dn[q] = v;
        if (a == b) dd[a] = (a < R) ? p.vtv[a * R + a] * v : 0.0;
    }
    __syncthreads();
    double sh2 = 0.0;
    for (int z = 0; z < R; ++z) sh2 += dd[z];
    sh2 = p.eps * sh2 / R;
#pragma unroll
    for (int q = 0; q < EPT; ++q) {
        const int e = tid + NT * q, a = e / RB, b = e % RB;
        double v = (a < R && b < R) ? p.vtv[a * R + b] * dn[q] : (a == b ? 1.0 : 0.0);
        if (a == b && a < R) v += sh2;
        M[a * LDM + b] = v;
    }
    ok = cta_sweep<RB>(M);
    double wr = 0.0;
    if (tid < R) {
        for (int z = 0; z < R; ++z) wr = fma(-M[tid * LDM + z], cv[z], wr);
        ok = ok && isfinite(wr);
    }
    if (!__syncthreads_and(ok)) {
        if (tid == 0) atomicAdd(p.fallbacks, 1u);
#pragma unroll
        for (int q = 0; q < EPT; ++q) {
            const int e = tid + NT * q, a = e / RB, b = e % RB;
            double v = (a < R && b < R) ? p.vtv[a * R + b] * dn[q] : (a == b ? 1.0 : 0.0);
            if (a == b && a < R) v += sh2;
            M[a * LDM + b] = v;
        }
        __syncthreads();
        if (!cta_lu_neg_inverse<RB>(M, piv, R, red) && tid == 0) report_error(p.err, m, DASH_E_SINGULAR);
        wr = 0.0;
        if (tid < R) {
            for (int z = 0; z < R; ++z) wr = fma(-M[tid * LDM + z], cv[z], wr);
            if (!isfinite(wr)) report_error(p.err, m, DASH_E_NONFINITE);
        }
    }
    if (tid < RB) wv[tid] = tid < R ? wr : 0.0;
    if (tid < R) {
        p.W[(int64_t)wrow * R + tid] = wr;
        if (p.final_pass) p.C[(int64_t)wrow * R + tid] = cv[tid];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < EPT; ++q) {
        const int e = tid + NT * q, a = e / RB, b = e % RB;
        if (p.final_pass && a < R && b < R) p.D[(int64_t)wrow * R * R + a * R + b] = dn[q];
    }
    // ---- G contribution (one slice per CTA -> the item slot) and US rows
    double *slot = p.G_slots + (int64_t)blockIdx.x * R * R;
#pragma unroll
    for (int q = 0; q < EPT; ++q) {
        const int e = tid + NT * q, a = e / RB, b = e % RB;
        if (a < R && b < R) slot[a * R + b] = gram[q] * wv[a] * wv[b];
    }
    if (p.US != nullptr)
        for (int64_t e = tid; e < n * R; e += NT) p.US[r0 * R + e] = p.U[r0 * R + e] * wv[e % R];
}

// Finish one pass for large ranks (stream.py:344-346): every CTA forms
// G = sym(lam G0 + g), inverts it by the sweep (-> -G^-1, LU fallback) and
// writes its 32 rows of F = lam F0 + f and V = F G^-1.
template <int RB>
__global__ void __launch_bounds__(256) k_vsolve_cta(const double *__restrict__ fg, const double *__restrict__ F_snap,
                                                   const double *__restrict__ G_snap, double lam, int J, int R,
                                                   double eps, double *__restrict__ F, double *__restrict__ G,
                                                   double *__restrict__ V, unsigned long long *err,
                                                   unsigned int *fallbacks, const unsigned int *only_if = nullptr,
                                                   unsigned int gen = 0) {
    if (only_if != nullptr && *only_if != gen) return;  // k_vsolvew solved this update's V already
    using S = SC<RB>;
    constexpr int LDM = S::LDM;
    extern __shared__ double sm[];
    double *M = sm;
    double *red = M + RB * LDM;
    int *piv = reinterpret_cast<int *>(red + S::NT);
    const int tid = threadIdx.x;
    const int64_t JR = (int64_t)J * R;
    const double *g = fg + JR;
    for (int e = tid; e < RB * RB; e += S::NT) {
        const int a = e / RB, b = e % RB;
        double v = (a == b) ? 1.0 : 0.0;
        if (a < R && b < R) {
            const double m1 = lam * G_snap[a * R + b] + g[a * R + b];
            const double m2 = lam * G_snap[b * R + a] + g[b * R + a];
            v = (m1 + m2) / 2.0;
            if (blockIdx.x == 0) G[a * R + b] = v;
        }
        M[a * LDM + b] = v;
    }
    __syncthreads();
    double tr = 0.0;
    for (int z = 0; z < R; ++z) tr += M[z * LDM + z];
    const double sh = eps * (tr / R);
    __syncthreads();
    if (tid < R) M[tid * LDM + tid] += sh;
    bool ok = cta_sweep<RB>(M);
    if (!__syncthreads_and(ok)) {
        if (tid == 0 && blockIdx.x == 0) atomicAdd(fallbacks, 1u);
        for (int e = tid; e < RB * RB; e += S::NT) {
            const int a = e / RB, b = e % RB;
            double v = (a == b) ? 1.0 : 0.0;
            if (a < R && b < R) {
                const double m1 = lam * G_snap[a * R + b] + g[a * R + b];
                const double m2 = lam * G_snap[b * R + a] + g[b * R + a];
                v = (m1 + m2) / 2.0 + (a == b ? sh : 0.0);
            }
            M[a * LDM + b] = v;
        }
        __syncthreads();
        if (!cta_lu_neg_inverse<RB>(M, piv, R, red) && tid == 0) report_error(err, -1, DASH_E_SINGULAR);
    }
    // rows j0..j0+31 of F and V:  V[j][r] = sum_z F[j][z] (-M)[z][r]
    const int j0 = blockIdx.x * 32;
    __shared__ double Fs[32][RB];
    for (int e = tid; e < 32 * RB; e += S::NT) {
        const int jj = e / RB, z = e % RB, j = j0 + jj;
        double v = 0.0;
        if (j < J && z < R) {
            v = lam * F_snap[(int64_t)j * R + z] + fg[(int64_t)j * R + z];
            F[(int64_t)j * R + z] = v;
        }
        Fs[jj][z] = v;
    }
    __syncthreads();
    for (int e = tid; e < 32 * RB; e += S::NT) {
        const int jj = e / RB, r = e % RB, j = j0 + jj;
        if (j < J && r < R) {
            double v = 0.0;
            for (int z = 0; z < R; ++z) v = fma(-M[z * LDM + r], Fs[jj][z], v);
            V[(int64_t)j * R + r] = v;
            if (!isfinite(v)) report_error(err, -1, DASH_E_NONFINITE);
        }
    }
}
