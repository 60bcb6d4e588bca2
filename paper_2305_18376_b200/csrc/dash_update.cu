// DASH per-update step on B200 (sm_100a), FP64.
//
// Reference being replaced: StreamState.update (stream.py:251-370) and its
// numba kernel group_update (_kernels.py:62-144), paths under
// /root/reference/pkg/src/p2stream.  One update = `passes` x
//
//   k_prologue   vtv = V^T V; snapshots of F, G (pass 0); v_used (last pass)
//   k_xv         XV = X V                       (ragged-agnostic tall-skinny
//                                                GEMM on FP64 DMMA tensor cores)
//   k_slices     per slice: U = (XV o s) A^-1, c/D accumulation, W solve,
//                G contribution  (warp-per-slice, CTA-per-big-slice; the two
//                R x R ridge systems via warp Cholesky, LU fallback)
//   k_fgemm      F partials = X^T (U o w_slice(row))   (DMMA, split over rows)
//   colsum       fresh terms f, g = sums of the slots (fixed two-level order)
//   k_vsolve     F = lam F_snap + f, G = sym(lam G_snap + g), V = ridge_solve(G, F^T)^T
//
// All reductions use a fixed order (per-CTA slots summed in slot order), so
// results are bit-reproducible run to run, as the reference's determinism
// criterion requires (test_acceptance.py:416-475).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <mutex>
#include <type_traits>
#include <vector>

#include "../../include/dash_b200.h"
#include "dash_common.cuh"

using namespace dash;

namespace {

constexpr int kSmallRows = 32;     // slices with more rows are "big" (k_bigx / k_big)
constexpr int kSlicesPerItem = 16; // small slices grouped per CTA
constexpr int kFSplitRows = 1024;  // target rows per F-GEMM split

__host__ __device__ inline int rank_bucket(int R) {
    return R <= 4 ? 4 : R <= 8 ? 8 : R <= 16 ? 16 : R <= 32 ? 32 : 64;
}

// ---------------------------------------------------------------------------
// k_prologue: vtv, snapshots.  Blocks [0, nvb): vtv, one warp per (r, z)
// entry (lanes stride J in two interleaved chains, fixed-order shuffle tree:
// deterministic, and vtv[r][z] == vtv[z][r] bitwise since the products
// commute); the remaining blocks copy the snapshots.
// ---------------------------------------------------------------------------
constexpr int kVtvWarps = 8;  // vtv entries per block
__global__ void k_prologue(const double *__restrict__ V, int J, int R, double *__restrict__ vtv,
                           const double *__restrict__ F, const double *__restrict__ G,
                           double *__restrict__ F_snap, double *__restrict__ G_snap,
                           double *__restrict__ v_used, int snap, int last, int nvb) {
    if (blockIdx.x < nvb) {
        const int p = blockIdx.x * kVtvWarps + (threadIdx.x >> 5), lane = threadIdx.x & 31;
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
            if (lane == 0) vtv[p] = acc;
        }
        return;
    }
    const int tid = (blockIdx.x - nvb) * blockDim.x + threadIdx.x, nt = (gridDim.x - nvb) * blockDim.x;
    if (snap) {
        for (int i = tid; i < J * R; i += nt) F_snap[i] = F[i];
        for (int i = tid; i < R * R; i += nt) G_snap[i] = G[i];
    }
    if (last)
        for (int i = tid; i < J * R; i += nt) v_used[i] = V[i];
}

// row -> batch position of its slice
__global__ void k_row_slice(const int64_t *__restrict__ row_ptr, int M, int32_t *__restrict__ row_slice) {
    int warps = (gridDim.x * blockDim.x) >> 5;
    int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    for (int m = gw; m < M; m += warps) {
        int64_t a = row_ptr[m], b = row_ptr[m + 1];
        for (int64_t r = a + lane_id(); r < b; r += 32) row_slice[r] = m;
    }
}

// US = U o w(slice of the row): the tensor-map F GEMM's operand when the slice kernel
// (k_slicesw) does not write it itself.  One element per thread, W rows from L2.
__global__ void k_us_rows(const double *__restrict__ U, const int32_t *__restrict__ row_slice,
                          const int32_t *__restrict__ state_row, const double *__restrict__ W, int R, int64_t n,
                          double *__restrict__ US) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i / R;
        const int r = (int)(i - row * R);
        US[i] = U[i] * W[(int64_t)state_row[row_slice[row]] * R + r];
    }
}

// ---------------------------------------------------------------------------
// k_xv: XV (N x R) = X (N x J, ld ldx) . V (J x R).  64-row tiles, 8 warps,
// warp w owns rows 8w..8w+7 of the tile and all RP/8 column tiles.
// ---------------------------------------------------------------------------
template <int RP, typename TX>
__global__ void __launch_bounds__(256) k_xv(const TX *__restrict__ X, int64_t ldx, int64_t N, int J,
                                            const double *__restrict__ V, int R, double *__restrict__ XV) {
    constexpr int BM = 64, BK = 32, LDXS = BK + 4;
    constexpr int LDVS = (RP % 16 == 0) ? RP + 8 : RP;
    constexpr int NT = RP / 8;
    __shared__ double Xs[BM * LDXS];
    __shared__ double Vs[BK * LDVS];
    const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
    const int g = lane >> 2, t = lane & 3;
    const int64_t ntiles = (N + BM - 1) / BM;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t row0 = tile * BM;
        double acc[NT][2];
#pragma unroll
        for (int n = 0; n < NT; ++n) acc[n][0] = acc[n][1] = 0.0;
        for (int k0 = 0; k0 < J; k0 += BK) {
#pragma unroll
            for (int q = 0; q < (BM * BK) / 256; ++q) {
                int i = tid + q * 256;
                int r = i / BK, c = i % BK;
                int64_t row = row0 + r;
                int col = k0 + c;
                Xs[r * LDXS + c] = (row < N && col < J) ? (double)__ldg(X + row * ldx + col) : 0.0;
            }
            for (int i = tid; i < BK * RP; i += 256) {
                int r = i / RP, c = i % RP;
                int jj = k0 + r;
                Vs[r * LDVS + c] = (jj < J && c < R) ? __ldg(V + jj * R + c) : 0.0;
            }
            __syncthreads();
#pragma unroll
            for (int kk = 0; kk < BK / 4; ++kk) {
                double a = Xs[(w * 8 + g) * LDXS + kk * 4 + t];
#pragma unroll
                for (int n = 0; n < NT; ++n) {
                    double b = Vs[(kk * 4 + t) * LDVS + n * 8 + g];
                    dmma884(acc[n], a, b);
                }
            }
            __syncthreads();
        }
        const int64_t row = row0 + w * 8 + g;
        if (row < N) {
#pragma unroll
            for (int n = 0; n < NT; ++n)
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    int col = n * 8 + t * 2 + i;
                    if (col < R) XV[row * R + col] = acc[n][i];
                }
        }
    }
}

// ---------------------------------------------------------------------------
// k_slices: the per-slice phase (_kernels.py:62-144 semantics).
// ---------------------------------------------------------------------------
struct SliceParams {
    const int4 *items;          // {slice0, nslices, big, 0}
    const int64_t *row_ptr;
    const int32_t *state_row;
    const uint8_t *is_new;
    const double *XV;           // N x R
    double *U;                  // N x R
    double *US;                 // N x R: U o w_slice (F-GEMM operand), may be null
    double *W, *C, *D;          // state rows
    const double *vtv;          // R x R
    double *G_slots;            // nitems x R x R
    unsigned long long *err;
    unsigned int *fallbacks;    // count of systems that needed LU
    int R;
    double lam, eps;
    int pass, final_pass;
    int sweep_only = 0;         // k_slices3: exact sweep for every A system (no Neumann fast path)
};

template <int RB>
struct SliceSmem {
    static constexpr int LD = RB + 1;
    static constexpr int NP = RB * (RB + 1) / 2;  // gram pairs (upper triangle)
    static constexpr int NPC = NP + RB;           // + the R entries of c
    // per warp: L[RB*LD] | Us[32*LD] | Xs[32*LD] | gram[RB*LD] | dinv | svec | vec | piv
    static constexpr int per_warp = RB * LD + 32 * LD + 32 * LD + RB * LD + 4 * RB;
    __host__ __device__ static constexpr int shared(int nw) { return RB * LD + 2 * NPC + nw * NPC; }
    __host__ __device__ static constexpr size_t bytes(int nw) {
        return sizeof(double) * (shared(nw) + nw * per_warp);
    }
};

// Pair index p -> (r, z).  p < NP: gram entry (r <= z, row-major upper
// triangle); NP <= p < NP + RB: the c entry r = z = p - NP.
__device__ __forceinline__ void pair_rz(int p, int RB, int &r, int &z) {
    const int NP = RB * (RB + 1) / 2;
    if (p >= NP) { r = z = p - NP; return; }
    int rr = 0, base = 0;
    while (p >= base + (RB - rr)) { base += RB - rr; ++rr; }
    r = rr;
    z = rr + (p - base);
}

template <int RB, int NW>
__global__ void __launch_bounds__(NW * 32) k_slices(SliceParams p) {
    using S = SliceSmem<RB>;
    constexpr int LD = S::LD, NP = S::NP, NPC = S::NPC, NPL = (NPC + 31) / 32;
    extern __shared__ double sm[];
    double *vtv_s = sm;                               // RB x LD
    int *pr_s = reinterpret_cast<int *>(vtv_s + RB * LD);  // NPC ints (stored in 2*NPC doubles)
    int *pz_s = pr_s + NPC;
    double *red = vtv_s + RB * LD + 2 * NPC;          // NW x NPC
    const int lane = lane_id(), w = warp_id();
    double *wbase = sm + S::shared(NW) + w * S::per_warp;
    double *Ls = wbase;
    double *Us = Ls + RB * LD;
    double *Xs = Us + 32 * LD;
    double *gram_s = Xs + 32 * LD;
    double *dinv = gram_s + RB * LD;
    double *svec = dinv + RB;
    double *vec = svec + RB;
    int *piv = reinterpret_cast<int *>(vec + RB);

    const int R = p.R;
    for (int i = threadIdx.x; i < RB * LD; i += blockDim.x) {
        int r = i / LD, z = i % LD;
        vtv_s[i] = (r < R && z < R) ? p.vtv[r * R + z] : 0.0;
    }
    for (int i = threadIdx.x; i < NPC; i += blockDim.x) {
        int r, z;
        pair_rz(i, RB, r, z);
        pr_s[i] = r;
        pz_s[i] = z;
    }
    __syncthreads();

    double g_loc[NPL];
#pragma unroll
    for (int q = 0; q < NPL; ++q) g_loc[q] = 0.0;

    const int4 item = p.items[blockIdx.x];
    const bool big = item.z != 0;
    const int nsl = item.y;

    for (int si = big ? 0 : w; si < nsl; si += big ? nsl : NW) {
        const int m = item.x + si;
        const int64_t r0 = p.row_ptr[m], r1 = p.row_ptr[m + 1];
        const int wrow = p.state_row[m];
        const bool fresh = p.is_new[m] != 0;
        if (lane < RB)
            svec[lane] = (lane < R) ? ((fresh && p.pass == 0) ? 1.0 : p.W[(int64_t)wrow * R + lane]) : 0.0;
        __syncwarp();

        // ---- row-factor system A = vtv o s s^T + shift I (_kernels.py:86-97)
        double sh = 0.0;
        for (int r = 0; r < R; ++r) sh += vtv_s[r * LD + r] * svec[r] * svec[r];
        sh = p.eps * sh / R;
        bool cholA;
        {
            double row[RB];
            const double sl = lane < RB ? svec[lane] : 0.0;
#pragma unroll
            for (int z = 0; z < RB; ++z) {
                double v = 0.0;
                if (lane < R && z < R) {
                    v = vtv_s[lane * LD + z] * sl * svec[z];
                    if (z == lane) v += sh;
                } else if (z == lane) {
                    v = 1.0;
                }
                row[z] = v;
            }
            cholA = chol_regs<RB>(row, Ls, LD, dinv);
        }
        if (!cholA) {
            // LU fallback on the unpadded system (stream.py:324-329 -> np.linalg.solve)
            if (lane == 0) {
                atomicAdd(p.fallbacks, 1u);
                for (int r = 0; r < R; ++r)
                    for (int z = 0; z < R; ++z)
                        Ls[r * LD + z] = vtv_s[r * LD + z] * svec[r] * svec[z] + (r == z ? sh : 0.0);
                if (!lu_factor_serial(Ls, LD, R, piv)) report_error(p.err, m, DASH_E_SINGULAR);
            }
            __syncwarp();
        }

        // ---- rows: U, then c / gram partials from the staged rows
        double gp[NPL];
#pragma unroll
        for (int q = 0; q < NPL; ++q) gp[q] = 0.0;
        const int64_t nrows = r1 - r0;
        const int nchunks = (int)((nrows + 31) / 32);
        for (int ch = big ? w : 0; ch < nchunks; ch += big ? NW : 1) {
            const int64_t row = r0 + (int64_t)ch * 32 + lane;
            const bool valid = row < r1;
            double b[RB];
#pragma unroll
            for (int r = 0; r < RB; ++r) {
                double x = (valid && r < R) ? p.XV[row * R + r] : 0.0;
                Xs[lane * LD + r] = x;
                b[r] = x * svec[r];
            }
            if (cholA) {
                chol_solve_lane<RB>(Ls, LD, dinv, b);
            } else {
                double *scr = Us + lane * LD;
                
#pragma unroll
                for (int r = 0; r < RB; ++r) if (r < R) scr[r] = b[r];
                if (valid) lu_solve_serial(Ls, LD, R, piv, scr);
#pragma unroll
                for (int r = 0; r < RB; ++r) b[r] = (r < R) ? scr[r] : 0.0;
            }
#pragma unroll
            for (int r = 0; r < RB; ++r) {
                if (!valid) b[r] = 0.0;
                Us[lane * LD + r] = b[r];
            }
#pragma unroll
            for (int r = 0; r < RB; ++r)
                if (valid && r < R) p.U[row * R + r] = b[r];
            __syncwarp();
            // rows of this chunk that exist (the rest of Us / Xs is zero): short slices
            // skip the empty rows of the chunk instead of 32 FMAs per pair
            const int64_t left = r1 - (r0 + (int64_t)ch * 32);
            const int nv = left < 32 ? (int)left : 32;
#pragma unroll
            for (int q = 0; q < NPL; ++q) {
                const int pp = lane + 32 * q;
                if (pp < NPC) {
                    const int a = pr_s[pp], c = pz_s[pp];
                    const double *A = (pp < NP) ? Us : Xs;
                    double acc = gp[q];
#pragma unroll 4
                    for (int i = 0; i < nv; ++i) acc = fma(A[i * LD + a], Us[i * LD + c], acc);
                    gp[q] = acc;
                }
            }
            __syncwarp();
        }

        bool owner = true;
        if (big) {
            // combine the NW warps' partials in warp order
            double *mine = red + w * NPC;
#pragma unroll
            for (int q = 0; q < NPL; ++q)
                if (lane + 32 * q < NPC) mine[lane + 32 * q] = gp[q];
            __syncthreads();
            owner = (w == 0);
            if (owner) {
#pragma unroll
                for (int q = 0; q < NPL; ++q) {
                    int pp = lane + 32 * q;
                    if (pp < NPC) {
                        double acc = 0.0;
                        for (int ww = 0; ww < NW; ++ww) acc += red[ww * NPC + pp];
                        gp[q] = acc;
                    }
                }
            }
        }

        if (owner) {
            // gram (symmetric) and c to shared
#pragma unroll
            for (int q = 0; q < NPL; ++q) {
                const int pp = lane + 32 * q;
                if (pp < NP) {
                    gram_s[pr_s[pp] * LD + pz_s[pp]] = gp[q];
                    gram_s[pz_s[pp] * LD + pr_s[pp]] = gp[q];
                } else if (pp < NPC) {
                    vec[pp - NP] = gp[q];
                }
            }
            __syncwarp();
            // ---- c, D accumulation and the S-row system (_kernels.py:103-135)
            double *dn = Us;  // reuse as d_new (RB x LD)
            for (int i = lane; i < RB * RB; i += 32) {
                int r = i / RB, z = i % RB;
                double v = 0.0;
                if (r < R && z < R) {
                    double dold = fresh ? 0.0 : p.D[(int64_t)wrow * R * R + r * R + z];
                    v = p.lam * dold + gram_s[r * LD + z];
                }
                dn[r * LD + z] = v;
            }
            double cn = 0.0;
            if (lane < R) {
                double cold = fresh ? 0.0 : p.C[(int64_t)wrow * R + lane];
                cn = p.lam * cold + vec[lane];
            }
            __syncwarp();
            double sh2 = 0.0;
            for (int r = 0; r < R; ++r) sh2 += vtv_s[r * LD + r] * dn[r * LD + r];
            sh2 = p.eps * sh2 / R;
            double wv;
            bool cholB;
            {
                double row[RB];
#pragma unroll
                for (int z = 0; z < RB; ++z) {
                    double v = 0.0;
                    if (lane < R && z < R) {
                        v = vtv_s[lane * LD + z] * dn[lane * LD + z];
                        if (z == lane) v += sh2;
                    } else if (z == lane) {
                        v = 1.0;
                    }
                    row[z] = v;
                }
                cholB = chol_regs<RB>(row, Ls, LD, dinv);
                wv = chol_solve_dist<RB>(row, Ls, LD, dinv, cn);
            }
            bool fin = (lane >= R) || finite_d(wv);
            bool good = cholB && __all_sync(FULL_MASK, fin);
            if (!good) {
                if (lane == 0) {
                    atomicAdd(p.fallbacks, 1u);
                    for (int r = 0; r < R; ++r)
                        for (int z = 0; z < R; ++z)
                            Ls[r * LD + z] = vtv_s[r * LD + z] * dn[r * LD + z] + (r == z ? sh2 : 0.0);
                    if (!lu_factor_serial(Ls, LD, R, piv)) report_error(p.err, m, DASH_E_SINGULAR);
                }
                __syncwarp();
                if (lane < R) vec[lane] = cn;
                __syncwarp();
                if (lane == 0) {
                    lu_solve_serial(Ls, LD, R, piv, vec);
                    for (int r = 0; r < R; ++r)
                        if (!finite_d(vec[r])) { report_error(p.err, m, DASH_E_NONFINITE); break; }
                }
                __syncwarp();
                wv = (lane < R) ? vec[lane] : 0.0;
            }
            if (lane < R) {
                p.W[(int64_t)wrow * R + lane] = wv;
                if (p.final_pass) p.C[(int64_t)wrow * R + lane] = cn;
            }
            if (p.final_pass)
                for (int i = lane; i < R * R; i += 32)
                    p.D[(int64_t)wrow * R * R + i] = dn[(i / R) * LD + (i % R)];
            __syncwarp();
            if (lane < RB) vec[lane] = (lane < R) ? wv : 0.0;
            __syncwarp();
            // ---- G contribution: gram o w w^T (_kernels.py:139-143)
#pragma unroll
            for (int q = 0; q < NPL; ++q) {
                const int pp = lane + 32 * q;
                if (pp < NP) g_loc[q] = fma(gp[q] * vec[pr_s[pp]], vec[pz_s[pp]], g_loc[q]);
            }
            __syncwarp();
        }
        if (big) __syncthreads();
    }

    // ---- per-item G slot: sum warps in order
    __syncthreads();
    {
        double *mine = red + w * NPC;
#pragma unroll
        for (int q = 0; q < NPL; ++q)
            if (lane + 32 * q < NPC) mine[lane + 32 * q] = g_loc[q];
    }
    __syncthreads();
    double *slot = p.G_slots + (int64_t)blockIdx.x * R * R;
    for (int pp = threadIdx.x; pp < NP; pp += blockDim.x) {
        double acc = 0.0;
        for (int ww = 0; ww < NW; ++ww) acc += red[ww * NPC + pp];
        const int r = pr_s[pp], z = pz_s[pp];
        if (r < R && z < R) {
            slot[r * R + z] = acc;
            slot[z * R + r] = acc;
        }
    }
}

// Kernel launch, optionally with programmatic stream serialization (PDL):
// only for kernels that call pdl_wait() before touching their predecessor's
// data (dash_common.cuh).  DASH_NO_PDL=1 disables it (A/B timing).
// Raise a kernel's dynamic shared-memory limit once (not on every update):
// keyed by (kernel address, current device): the attribute is per device, so
// a second GPU in the same process gets its own opt-in.  Thread-safe.
struct SmemAttrKey {
    const void *kern;
    int dev;
    size_t smem;
};
template <typename K>
void ensure_smem_attr(K kern, size_t smem) {
    static std::mutex mu;
    static std::vector<SmemAttrKey> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    const void *key = reinterpret_cast<const void *>(kern);
    for (auto &e : done)
        if (e.kern == key && e.dev == dev) {
            if (e.smem < smem) {
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                e.smem = smem;
            }
            return;
        }
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    done.push_back({key, dev, smem});
}

bool pdl_enabled() {
    static const bool on = getenv("DASH_NO_PDL") == nullptr;
    return on;
}
// per-launch-site switch for A/B timing: DASH_PDL_OFF=<comma list of site names>
bool pdl_site(const char *name) {
    static const char *off = getenv("DASH_PDL_OFF");
    return !(off && strstr(off, name));
}

template <typename... KArgs, typename... Args>
int launch_k(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = (pdl && pdl_enabled()) ? 1 : 0;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, args...);
    if (e != cudaSuccess) {
        static const bool verbose = getenv("DASH_VERBOSE") != nullptr;
        if (verbose)
            fprintf(stderr, "[dash] launch failed: %s (grid %u, block %u, smem %zu)\n", cudaGetErrorString(e), grid.x,
                    block.x, smem);
        return DASH_E_CUDA;
    }
    return 0;
}

#include "dash_slices.cuh"
#include "dash_stream.cuh"
#include "dash_tma.cuh"
#include "dash_tma32.cuh"
#include "dash_slices_cta.cuh"
#include "dash_slices3.cuh"
#include "dash_big.cuh"
#include "dash_bigx.cuh"
#include "dash_smallx.cuh"
#include "dash_slicesw.cuh"
#include "dash_widej.cuh"

// ---------------------------------------------------------------------------
// k_fgemm: F partial slot s = X[rows_s]^T (U o w)[rows_s], J-block of 64.
// ---------------------------------------------------------------------------
template <int RP, typename TX>
__global__ void __launch_bounds__(256) k_fgemm(const TX *__restrict__ X, int64_t ldx, int64_t N, int J,
                                               const double *__restrict__ U, const int32_t *__restrict__ row_slice,
                                               const int32_t *__restrict__ state_row, const double *__restrict__ W,
                                               int R, int64_t rows_per_split, double *__restrict__ F_slots,
                                               double *__restrict__ G_slots) {
    // G_slots != null: the last column block computes US^T US (G's fresh term,
    // sum_k gram_k o w_k w_k^T of _kernels.py:139-143 summed by rows) instead of X^T US
    constexpr int BJ = 64, BK = 32, LDXS = BJ + 8;
    constexpr int LDUS = (RP % 16 == 0) ? RP + 8 : RP;
    constexpr int NT = RP / 8;
    __shared__ double Xs[BK * LDXS];
    __shared__ double Ss[BK * LDUS];
    const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
    const int g = lane >> 2, t = lane & 3;
    const bool gblk = G_slots != nullptr && blockIdx.x == gridDim.x - 1;
    const int j0 = gblk ? 0 : blockIdx.x * BJ;
    const int64_t rbeg = (int64_t)blockIdx.y * rows_per_split;
    const int64_t rend = min(N, rbeg + rows_per_split);
    double acc[NT][2];
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[n][0] = acc[n][1] = 0.0;
    for (int64_t k0 = rbeg; k0 < rend; k0 += BK) {
#pragma unroll
        for (int q = 0; q < (BK * BJ) / 256; ++q) {
            int i = tid + q * 256;
            int r = i / BJ, c = i % BJ;
            int64_t row = k0 + r;
            int col = j0 + c;
            if (gblk) {
                double v = 0.0;
                if (row < rend && c < R)
                    v = U[row * R + c] * W[(int64_t)state_row[row_slice[row]] * R + c];
                Xs[r * LDXS + c] = v;
            } else {
                Xs[r * LDXS + c] = (row < rend && col < J) ? (double)__ldg(X + row * ldx + col) : 0.0;
            }
        }
        for (int i = tid; i < BK * RP; i += 256) {
            int r = i / RP, c = i % RP;
            int64_t row = k0 + r;
            double v = 0.0;
            if (row < rend && c < R) {
                int m = row_slice[row];
                v = U[row * R + c] * W[(int64_t)state_row[m] * R + c];
            }
            Ss[r * LDUS + c] = v;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK / 4; ++kk) {
            double a = Xs[(kk * 4 + t) * LDXS + w * 8 + g];
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                double b = Ss[(kk * 4 + t) * LDUS + n * 8 + g];
                dmma884(acc[n], a, b);
            }
        }
        __syncthreads();
    }
    double *slot = gblk ? G_slots + (int64_t)blockIdx.y * R * R : F_slots + (int64_t)blockIdx.y * J * R;
    const int j = j0 + w * 8 + g;
    if (j < (gblk ? R : J)) {
#pragma unroll
        for (int n = 0; n < NT; ++n)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                int col = n * 8 + t * 2 + i;
                if (col < R) slot[j * R + col] = acc[n][i];
            }
    }
}

// Column sums of a (nslots x width) slot matrix in fixed order, two levels:
// k_colsum_part sums segments of kSeg slots, k_colsum_final sums segments.
// Used for fg = [sum F slots | sum G slots] (the fresh terms f_fresh, g_fresh
// of stream.py:306-322; raw, not yet decayed).
constexpr int kSeg = 32;

__global__ void k_colsum_part(const double *__restrict__ slots, int nslots, int64_t width,
                              double *__restrict__ part) {
    const int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int seg = blockIdx.y;
    if (col >= width) return;
    const int s0 = seg * kSeg, s1 = min(nslots, s0 + kSeg);
    double acc = 0.0;
    for (int s = s0; s < s1; ++s) acc += slots[(int64_t)s * width + col];
    part[(int64_t)seg * width + col] = acc;
}

__global__ void k_colsum_final(const double *__restrict__ part, int nseg, int64_t width,
                               double *__restrict__ out) {
    const int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= width) return;
    double acc = 0.0;
    for (int s = 0; s < nseg; ++s) acc += part[(int64_t)s * width + col];
    out[col] = acc;
}

// Two slot arrays (F and G) summed by one pair of launches: blocks [0, a.nblk)
// serve job a, the rest job b.  Same fixed segment order as k_colsum_part /
// k_colsum_final (deterministic); loads unrolled so a segment's slots are in flight.
struct ColSumJob {
    const double *slots;
    double *part, *out;
    int64_t width;
    int nslots, nseg, bx;
};

__global__ void __launch_bounds__(128) k_colsum_part2(ColSumJob a, ColSumJob b) {
    pdl_wait();
    pdl_trigger();
    int blk = blockIdx.x;
    const bool second = blk >= a.bx * a.nseg;
    const ColSumJob &j = second ? b : a;
    if (second) blk -= a.bx * a.nseg;
    const int64_t col = (int64_t)(blk % j.bx) * blockDim.x + threadIdx.x;
    const int seg = blk / j.bx;
    if (col >= j.width) return;
    const int s0 = seg * kSeg, s1 = min(j.nslots, s0 + kSeg);
    double acc = 0.0;
    int s = s0;
    for (; s + 8 <= s1; s += 8) {
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = j.slots[(int64_t)(s + k) * j.width + col];
#pragma unroll
        for (int k = 0; k < 8; ++k) acc += v[k];
    }
    for (; s < s1; ++s) acc += j.slots[(int64_t)s * j.width + col];
    j.part[(int64_t)seg * j.width + col] = acc;
}

__global__ void __launch_bounds__(128) k_colsum_final2(ColSumJob a, ColSumJob b) {
    pdl_wait();
    pdl_trigger();
    int blk = blockIdx.x;
    const bool second = blk >= a.bx;
    const ColSumJob &j = second ? b : a;
    if (second) blk -= a.bx;
    const int64_t col = (int64_t)blk * blockDim.x + threadIdx.x;
    if (col >= j.width) return;
    double acc = 0.0;
    for (int s = 0; s < j.nseg; ++s) acc += j.part[(int64_t)s * j.width + col];
    j.out[col] = acc;
}

// Finish one pass (stream.py:344-346): F = lam F_snap + f, G = sym(lam G_snap
// + g), then V = ridge_solve(G, F^T)^T (linalg.py:25-45).  Every warp forms G
// and factors it (identical result in every warp) and solves 32 rows of V;
// block 0 / warp 0 writes G, each warp writes its F rows.
template <int RB, int NWV>
__global__ void __launch_bounds__(NWV * 32) k_vsolve(const double *__restrict__ fg, const double *__restrict__ F_snap,
                                                     const double *__restrict__ G_snap, double lam, int J, int R,
                                                     double eps, double *__restrict__ F, double *__restrict__ G,
                                                     double *__restrict__ V, unsigned long long *err,
                                                     unsigned int *fallbacks, const unsigned int *only_if = nullptr,
                                                     unsigned int gen = 0) {
    constexpr int LD = RB + 1;
    pdl_wait();
    pdl_trigger();
    if (only_if != nullptr && *only_if != gen) return;  // k_vsolvew solved this update's V already
    __shared__ double sL[NWV][RB * LD];
    __shared__ double sG[NWV][RB * LD];
    __shared__ double sd[NWV][RB];
    __shared__ int spiv[NWV][RB];
    __shared__ double sx[NWV][32][LD];
    const int lane = lane_id(), w = warp_id();
    double *Ls = sL[w], *Gs = sG[w], *dinv = sd[w];
    const int64_t JR = (int64_t)J * R;
    const double *g = fg + JR;
    for (int i = lane; i < R * R; i += 32) {
        const int r = i / R, z = i % R;
        const double m1 = lam * G_snap[r * R + z] + g[r * R + z];
        const double m2 = lam * G_snap[z * R + r] + g[z * R + r];
        Gs[r * LD + z] = (m1 + m2) / 2.0;
    }
    __syncwarp();
    if (blockIdx.x == 0 && w == 0)
        for (int i = lane; i < R * R; i += 32) G[i] = Gs[(i / R) * LD + (i % R)];
    double tr = 0.0;
    for (int r = 0; r < R; ++r) tr += Gs[r * LD + r];
    const double sh = eps * (tr / R);
    double row[RB];
#pragma unroll
    for (int z = 0; z < RB; ++z) {
        double v = 0.0;
        if (lane < R && z < R) {
            v = Gs[lane * LD + z];
            if (z == lane) v += sh;
        } else if (z == lane) {
            v = 1.0;
        }
        row[z] = v;
    }
    bool ok = chol_regs<RB>(row, Ls, LD, dinv);
    if (!ok) {
        if (lane == 0) {
            if (blockIdx.x == 0 && w == 0) atomicAdd(fallbacks, 1u);
            for (int r = 0; r < R; ++r)
                for (int z = 0; z < R; ++z) Ls[r * LD + z] = Gs[r * LD + z] + (r == z ? sh : 0.0);
            if (!lu_factor_serial(Ls, LD, R, spiv[w])) report_error(err, -1, DASH_E_SINGULAR);
        }
        __syncwarp();
    }
    const int j = (blockIdx.x * NWV + w) * 32 + lane;
    const bool valid = j < J;
    double b[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) {
        double v = 0.0;
        if (valid && r < R) {
            v = lam * F_snap[(int64_t)j * R + r] + fg[(int64_t)j * R + r];
            F[(int64_t)j * R + r] = v;
        }
        b[r] = v;
    }
    if (ok) {
        chol_solve_lane<RB>(Ls, LD, dinv, b);
    } else {
        double *scr = sx[w][lane];
#pragma unroll
        for (int r = 0; r < RB; ++r)
            if (r < R) scr[r] = b[r];
        if (valid) lu_solve_serial(Ls, LD, R, spiv[w], scr);
#pragma unroll
        for (int r = 0; r < RB; ++r) b[r] = (r < R) ? scr[r] : 0.0;
    }
    if (valid) {
        bool fin = true;
#pragma unroll
        for (int r = 0; r < RB; ++r) {
            if (r < R) {
                V[(int64_t)j * R + r] = b[r];
                fin = fin && finite_d(b[r]);
            }
        }
        if (!fin) report_error(err, -1, DASH_E_NONFINITE);
    }
}

// V solve for R <= 16 in ONE short chain: warp 0 forms G = sym(lam G0 + g)
// + shift I and inverts it with the unit-pivot sweep (A / max diag, LU with
// partial pivoting if a pivot fails -- the reference solves with LU,
// linalg.py:25-45), then every thread forms one row F_j = lam F0_j + f_j and
// V_j = G^{-1} F_j (16 x 16 FMAs against the broadcast inverse).  Replaces the
// per-warp Cholesky + per-lane triangular solves of k_vsolve (latency chain
// of 2 x 16 dependent steps per lane).
template <int RB>
__global__ void __launch_bounds__(128) k_vsolve2(const double *__restrict__ fg, const double *__restrict__ F_snap,
                                                 const double *__restrict__ G_snap, double lam, int J, int R,
                                                 double eps, double *__restrict__ F, double *__restrict__ G,
                                                 double *__restrict__ V, unsigned long long *err,
                                                 unsigned int *fallbacks) {
    constexpr int LDL = RB + 1, NGR = 32 / RB;
    __shared__ double gi[RB * LDL];                     // G^{-1}
    __shared__ __align__(16) double gbuf[NGR][RB + 2];  // one gather buffer per lane group
    __shared__ double lu[RB * LDL];
    __shared__ int piv[RB];
    pdl_wait();
    pdl_trigger();
    const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
    const int64_t JR = (int64_t)J * R;
    const double *g = fg + JR;
    if (w == 0) {
        const int r = lane % RB;
        const bool real = lane < RB && r < R;  // lanes >= RB: harmless identity systems
        // trace of sym(lam G0 + g): lane r holds entry (r, r); fixed-order reduction over lanes 0..R-1
        double tr = 0.0;
        {
            const double dr = (lane < R) ? lam * G_snap[lane * R + lane] + __ldcg(g + lane * R + lane) : 0.0;
            if (lane == 0) tr = dr;
            for (int z = 1; z < R; ++z) {  // same order as the serial sum (bit-identical)
                const double v = __shfl_sync(FULL_MASK, dr, z);
                if (lane == 0) tr += v;
            }
            tr = __shfl_sync(FULL_MASK, tr, 0);
        }
        const double sh = eps * (tr / R);
        double a[RB];
#pragma unroll
        for (int z = 0; z < RB; ++z) {
            double v = (z == r) ? 1.0 : 0.0;
            if (real && z < R) {
                const double m1 = lam * G_snap[r * R + z] + __ldcg(g + r * R + z);
                const double m2 = lam * G_snap[z * R + r] + __ldcg(g + z * R + r);
                v = (m1 + m2) / 2.0;
                if (blockIdx.x == 0) G[r * R + z] = v;
                if (z == r) v += sh;
            }
            a[z] = v;
        }
        double mx = 0.0;
#pragma unroll
        for (int z = 0; z < RB; ++z)
            if (z == r) mx = a[z];
#pragma unroll
        for (int off = RB / 2; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL_MASK, mx, off));
        double im = (mx > 0.0 && isfinite(mx)) ? 1.0 / mx : 1.0;
        double a0[RB];
#pragma unroll
        for (int z = 0; z < RB; ++z) {
            a0[z] = a[z];
            a[z] *= im;
        }
        const bool ok = __all_sync(FULL_MASK, sweep_inverse_unit<RB>(a, gbuf[lane / RB], r) || lane >= RB);
        if (!ok) {  // LU with partial pivoting on the unscaled system (lane 0 of group 0)
#pragma unroll
            for (int z = 0; z < RB; ++z) a[z] = a0[z];
            if (lane == 0 && blockIdx.x == 0) atomicAdd(fallbacks, 1u);
            const bool okLU = lu_fallback<RB>(a, lu, piv, r, R, lane < RB);
            if (lane == 0 && !okLU) report_error(err, -1, DASH_E_SINGULAR);
            im = 1.0;
        }
        if (lane < RB) {  // a = -(scaled G)^{-1}  ->  G^{-1} = -a / max diag
#pragma unroll
            for (int z = 0; z < RB; ++z) gi[r * LDL + z] = -a[z] * im;
        }
    }
    __syncthreads();
    const int j = blockIdx.x * blockDim.x + tid;
    if (j >= J) return;
    double fj[RB];
#pragma unroll
    for (int z = 0; z < RB; ++z) {
        double v = 0.0;
        if (z < R) {
            v = lam * F_snap[(int64_t)j * R + z] + __ldcg(fg + (int64_t)j * R + z);
            F[(int64_t)j * R + z] = v;
        }
        fj[z] = v;
    }
    bool fin = true;
#pragma unroll
    for (int r = 0; r < RB; ++r) {
        if (r < R) {
            double acc = 0.0;
#pragma unroll
            for (int z = 0; z < RB; ++z) acc = fma(gi[r * LDL + z], fj[z], acc);
            V[(int64_t)j * R + r] = acc;
            fin = fin && finite_d(acc);
        }
    }
    if (!fin) report_error(err, -1, DASH_E_NONFINITE);
}

// us = u o w  (group_update seam output)
__global__ void k_us(const double *__restrict__ u, const double *__restrict__ w, int G, int I, int R,
                     double *__restrict__ us) {
    int64_t n = (int64_t)G * I * R;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t g = i / ((int64_t)I * R);
        int r = (int)(i % R);
        us[i] = u[i] * w[g * R + r];
    }
}

// g_fresh = sum of item slots in order
__global__ void k_sum_slots(const double *__restrict__ slots, int n, int RR, double *__restrict__ out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < RR) {
        double acc = 0.0;
        for (int s = 0; s < n; ++s) acc += slots[(int64_t)s * RR + i];
        out[i] = acc;
    }
}

}  // namespace

// ===========================================================================
// host side
// ===========================================================================
namespace {
// F = lam F_snap + f, G = sym(lam G_snap + g)  (no V solve; init_helpers uses lam = 0)
__global__ void k_finish_fg(const double *__restrict__ fg, const double *__restrict__ F_snap,
                            const double *__restrict__ G_snap, double lam, int J, int R, double *__restrict__ F,
                            double *__restrict__ G) {
    const int64_t JR = (int64_t)J * R;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < JR) {
        F[i] = lam * F_snap[i] + fg[i];
    } else if (i < JR + R * R) {
        const int p = (int)(i - JR), r = p / R, z = p % R;
        const double m1 = lam * G_snap[r * R + z] + fg[JR + r * R + z];
        const double m2 = lam * G_snap[z * R + r] + fg[JR + z * R + r];
        G[p] = (m1 + m2) / 2.0;
    }
}
}  // namespace

enum Phase { PH_ROWSLICE = 0, PH_PROLOGUE, PH_XV, PH_SLICES, PH_FGEMM, PH_SUMFG, PH_VSOLVE, PH_BIG, PH_BIGPOST, PH_COUNT };

struct dash_ctx {
    struct Buf {
        void *p = nullptr;
        size_t cap = 0;
    };
    Buf xv, row_slice, items, gslots, fslots, vtv, fsnap, gsnap, fg, part, us, scratch, smeta, plan_hist, u64;
    Buf tflag, bx_ms, bx_toff, bx_parts;  // fused big-slice path
    Buf rerr;                             // per-row reconstruction errors (local_error, ALS loss)
    Buf sw_scr;                           // k_slicesw per-warp scratch (R in (16, 64])
    bool swide = false;                   // R > 16 on k_slicesw (G's fresh term from the F GEMM)
    unsigned long long *err = nullptr;
    unsigned int *fallbacks = nullptr;
    unsigned int *vs_flag = nullptr;  // k_vsolvew -> fallback V solve hand-off (holds the failing launch's generation)
    unsigned int vs_gen = 0;
    int4 *items_host[2] = {nullptr, nullptr};
    size_t items_host_cap[2] = {0, 0};
    cudaEvent_t staged[2] = {nullptr, nullptr};
    int cur = 0;
    // batch index staging ring (dash_stage_meta): caller-owned pinned / device blocks
    struct MetaSlot {
        uint8_t *pin = nullptr, *dev = nullptr;
        cudaEvent_t copied = nullptr, done = nullptr;
        bool copy_issued = false, upd_issued = false;
    };
    static constexpr int kMetaSlots = 4;
    MetaSlot mring[kMetaSlots];
    int mring_n = 0, mring_i = 0, mring_last = -1;
    size_t mring_cap = 0;
    cudaStream_t meta_stream = nullptr;
    // Device slice plan on the staging side stream: the plan of update t+1 (k_plan_*: a pure
    // function of the batch's index arrays, which arrive on that stream) runs while update t's
    // kernels still execute.  Its outputs (smeta, plan_hist, tflag + tgen) are double-buffered:
    // the fields above/below hold the current set, pset_alt the other one; pset_free fires when
    // the update that read the current set has been issued in full.
    struct PlanSet {
        Buf smeta, plan_hist, tflag;
        uint32_t tgen = 0;
        cudaEvent_t free_ev = nullptr;
        bool used = false;
    } pset_alt;
    cudaEvent_t pset_free = nullptr, plan_ev = nullptr;
    // second stream + fork / join events for independent kernel pairs (ALS polar: long || short slices)
    cudaStream_t aux_stream = nullptr;
    cudaEvent_t aux_fork = nullptr, aux_join = nullptr;
    bool pset_used = false, side_plan = false;
    int cur_pass = 0;
    int last_launches = 0;
    int num_sms = 148;
    // per-update plan, shared by the pass_begin calls of one update
    int nitems = 0;
    int64_t nsplit = 1, rps = 32;
    bool stream = false;  // TMA-ring GEMM path for this update
    bool tma = false;     // ... with tensor-map (swizzled box) copies: k_xv3 / k_fgemm3
    bool bigx = false;    // big slices on the fused single-read path (dash_bigx.cuh)
    bool wtma = false;    // wide-J tensor-map GEMMs (dash_widej.cuh): J > 128, FP64 batches
    int wnj = 1;          // ... column blocks of the wide F GEMM
    int bigx_nbig = 0, bigx_grid = 0;
    bool smallx = false;  // small slices on the fused single-kernel path (dash_smallx.cuh)
    bool planned = false; // the device slice plan ran for this update
    int sx_grid = 0;
    Buf sx_tmp, sx_units, sx_meta;  // planner: per-chunk units | compacted units | counts, choff, nunits, done
    uint32_t tgen = 0;  // generation of the small-tile marks
    void *plan_p = nullptr;  // SlicePlan of the update in flight
    // phase timing (bench): events around every launch when enabled
    int prof = 0;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_recs;
    size_t ev_used = 0;
};

namespace {

cudaEvent_t prof_event(dash_ctx *ctx) {
    if (ctx->ev_used == ctx->ev_pool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        ctx->ev_pool.push_back(e);
    }
    return ctx->ev_pool[ctx->ev_used++];
}

struct PhaseScope {
    dash_ctx *ctx;
    cudaStream_t st;
    int id;
    cudaEvent_t a = nullptr;
    // NVTX range per phase (host-side launch window; header-only NVTX3: a no-op unless a
    // tool such as nsys / ncu --nvtx is attached), named like bench.py's phase keys
    static const char *phase_name(int i) {
        static const char *const names[PH_COUNT] = {"dash:row_slice", "dash:prologue", "dash:xv",      "dash:slices", "dash:fgemm",
                                                    "dash:sum_fg",    "dash:vsolve",   "dash:big",     "dash:big_post"};
        return (i >= 0 && i < PH_COUNT) ? names[i] : "dash:?";
    }
    PhaseScope(dash_ctx *c, cudaStream_t s, int i) : ctx(c), st(s), id(i) {
        nvtxRangePushA(phase_name(i));
        if (ctx->prof) {
            a = prof_event(ctx);
            cudaEventRecord(a, st);
        }
        ctx->last_launches++;
    }
    ~PhaseScope() {
        if (ctx->prof) {
            cudaEvent_t b = prof_event(ctx);
            cudaEventRecord(b, st);
            ctx->ev_recs.push_back({id, {a, b}});
        }
        nvtxRangePop();
    }
};

int ensure(dash_ctx::Buf &b, size_t bytes) {
    if (b.cap >= bytes) return 0;
    if (b.p) cudaFree(b.p);
    size_t cap = std::max(bytes + bytes / 2, (size_t)256);
    if (cudaMalloc(&b.p, cap) != cudaSuccess) {
        b.p = nullptr;
        b.cap = 0;
        return DASH_E_CUDA;
    }
    b.cap = cap;
    return 0;
}

int stage_items(dash_ctx *ctx, cudaStream_t st, const std::vector<int4> &items) {
    int c = ctx->cur;
    ctx->cur ^= 1;
    cudaEventSynchronize(ctx->staged[c]);
    size_t need = items.size() * sizeof(int4);
    if (ctx->items_host_cap[c] < need) {
        if (ctx->items_host[c]) cudaFreeHost(ctx->items_host[c]);
        size_t cap = need + need / 2 + 64;
        if (cudaMallocHost((void **)&ctx->items_host[c], cap) != cudaSuccess) return DASH_E_CUDA;
        ctx->items_host_cap[c] = cap;
    }
    memcpy(ctx->items_host[c], items.data(), need);
    if (ensure(ctx->items, need)) return DASH_E_CUDA;
    cudaMemcpyAsync(ctx->items.p, ctx->items_host[c], need, cudaMemcpyHostToDevice, st);
    cudaEventRecord(ctx->staged[c], st);
    return 0;
}

// Host planning: contiguous batch positions -> CTA work items.
void plan_items(const int64_t *row_ptr, int M, std::vector<int4> &items, int per_item = kSlicesPerItem) {
    items.clear();
    int m = 0;
    while (m < M) {
        int64_t n = row_ptr[m + 1] - row_ptr[m];
        if (n > kSmallRows) {
            items.push_back(make_int4(m, 1, 1, 0));
            ++m;
            continue;
        }
        int start = m, cnt = 0;
        while (m < M && cnt < per_item && (row_ptr[m + 1] - row_ptr[m]) <= kSmallRows) {
            ++m;
            ++cnt;
        }
        items.push_back(make_int4(start, cnt, 0, 0));
    }
    // big (one-CTA, long) items first so they do not form the grid's tail
    std::stable_partition(items.begin(), items.end(), [](const int4 &it) { return it.z != 0; });
}

void plan_fsplit(dash_ctx *ctx, int64_t N, int J, int64_t &nsplit, int64_t &rps) {
    nsplit = std::max<int64_t>(1, std::min<int64_t>((N + kFSplitRows - 1) / kFSplitRows,
                                                    (int64_t)ctx->num_sms * 8 / ((J + 63) / 64) + 1));
    rps = (N + nsplit - 1) / nsplit;
    rps = std::max<int64_t>(32, (rps + 31) / 32 * 32);
    nsplit = N > 0 ? (N + rps - 1) / rps : 1;
}

template <int RB>
int launch_slices(dash_ctx *ctx, cudaStream_t st, int nitems, const SliceParams &sp) {
    constexpr int NW = (RB <= 16) ? 8 : 4;
    size_t smem = SliceSmem<RB>::bytes(NW);
    ensure_smem_attr(k_slices<RB, NW>, smem);
    PhaseScope ps(ctx, st, PH_SLICES);
    k_slices<RB, NW><<<nitems, NW * 32, smem, st>>>(sp);
    return cudaGetLastError() == cudaSuccess ? 0 : DASH_E_CUDA;
}

int slices_per_item(int RB) { return RB <= 16 ? 2 * S2<16>::NW * (32 / RB) : RB <= 32 ? kSlicesPerItem : 1; }

int dispatch_slices(dash_ctx *ctx, cudaStream_t st, int RB, int nitems, const SliceParams &sp) {
    if (RB <= 16) {
        PhaseScope ps(ctx, st, PH_SLICES);
        switch (RB) {
            case 4: return launch_slices2<4>(st, nitems, sp);
            case 8: return launch_slices2<8>(st, nitems, sp);
            default: return launch_slices2<16>(st, nitems, sp);
        }
    }
    if (RB == 64) {
        const size_t smem = SC<64>::bytes();
        ensure_smem_attr(k_slices_cta<64>, smem);
        PhaseScope ps(ctx, st, PH_SLICES);
        k_slices_cta<64><<<nitems, 256, smem, st>>>(sp);
        return cudaGetLastError() == cudaSuccess ? 0 : DASH_E_CUDA;
    }
    return launch_slices<32>(ctx, st, nitems, sp);
}

// Slice-phase plan.  R <= 16: the slice order is planned ON DEVICE
// (k_plan_*: small slices longest first, big slices by size class) and the
// persistent k_slices3 (G slots [0, g3)) reads its work list from there.  Big
// slices go to the persistent DMMA kernel k_big (RB == 16, R even; slots [g3,
// g3 + gbig)), else to k_slices2 items planned on the host (slots [g3, g3 +
// nbig)).  Larger ranks keep the host item list of k_slices / k_slices_cta.
struct SlicePlan {
    std::vector<int4> items;  // host-planned items (k_slices2 big items, or all items for RB > 16)
    int nbig = 0, g3 = 0, gbig = 0, nslots = 0;
    int64_t big_tiles = 0;  // 32-row tiles of the big slices (fused path grid split)
    bool split = false, big_dev = false;
    bool wide = false;      // RB > 16 on k_slicesw: items = slice order, 4 positions per int4
};

// A/B switch: DASH_OLD_WIDE=1 keeps R > 16 on k_slices / k_slices_cta
bool wide_kernel() {
    static const bool v = getenv("DASH_OLD_WIDE") == nullptr;
    return v;
}

// Big-slice statistics of the last row_ptr built by dash_host_row_ptr on this
// thread: the planner reuses them instead of re-scanning row_ptr (M entries).
struct RowPtrStats {
    const int64_t *row_ptr = nullptr;
    int64_t M = -1, N = -1, tiles = 0;
    int nbig = 0;
};
thread_local RowPtrStats g_rp_stats;

SlicePlan make_plan(const int64_t *row_ptr, int M, int RB, int R, int num_sms) {
    SlicePlan pl;
    if (RB > 16 && wide_kernel()) {
        // k_slicesw order: multi-chunk slices first, longest first (stable), then the rest in
        // batch order; the warps take it strided, so the long solves start in the first wave
        std::vector<int32_t> ord;
        ord.reserve(M);
        for (int m = 0; m < M; ++m)
            if (row_ptr[m + 1] - row_ptr[m] > kSmallRows) ord.push_back(m);
        std::stable_sort(ord.begin(), ord.end(), [row_ptr](int a, int b) {
            return row_ptr[a + 1] - row_ptr[a] > row_ptr[b + 1] - row_ptr[b];
        });
        for (int m = 0; m < M; ++m)
            if (row_ptr[m + 1] - row_ptr[m] <= kSmallRows) ord.push_back(m);
        pl.items.assign((M + 3) / 4, make_int4(0, 0, 0, 0));
        if (M) memcpy(pl.items.data(), ord.data(), sizeof(int32_t) * M);
        pl.wide = true;
        return pl;
    }
    if (RB > 16) {
        plan_items(row_ptr, M, pl.items, slices_per_item(RB));
        pl.nslots = (int)pl.items.size();
        return pl;
    }
    pl.split = true;
    pl.g3 = kS3CtasPerSM * num_sms;
    if (RB == 16 && (R % 2) == 0) {  // order on device; the host only counts big slices (grid size)
        pl.big_dev = true;
        int nbig = 0;
        int64_t tiles = 0;
        const RowPtrStats &c = g_rp_stats;
        if (c.row_ptr == row_ptr && c.M == M && c.N == row_ptr[M]) {
            nbig = c.nbig;
            tiles = c.tiles;
        } else {
            for (int m = 0; m < M; ++m) {
                const int64_t n = row_ptr[m + 1] - row_ptr[m];
                if (n > kSmallRows) {
                    ++nbig;
                    tiles += (n + kTR - 1) / kTR;
                }
            }
        }
        pl.gbig = nbig;  // one CTA (and G slot) per big slice
        pl.big_tiles = tiles;
        pl.nslots = pl.g3 + pl.gbig;
        return pl;
    }
    for (int m = 0; m < M; ++m)
        if (row_ptr[m + 1] - row_ptr[m] > kSmallRows) pl.items.push_back(make_int4(m, 1, 1, 0));
    // longest first: one CTA per big slice -> shorter tail (stable: deterministic slot order)
    std::stable_sort(pl.items.begin(), pl.items.end(), [row_ptr](const int4 &a, const int4 &b) {
        return row_ptr[a.x + 1] - row_ptr[a.x] > row_ptr[b.x + 1] - row_ptr[b.x];
    });
    pl.nbig = (int)pl.items.size();
    pl.nslots = pl.g3 + pl.nbig;
    return pl;
}

SlicePlan &plan_of(dash_ctx *ctx) { return *reinterpret_cast<SlicePlan *>(ctx->plan_p); }

// device plan (R <= 16): meta[M] in plan order + plan_counts {nsmall, nbig}
template <class B>
int device_plan(dash_ctx *ctx, cudaStream_t st, const B *b, uint32_t *tflag) {
    const int M = b->M;
    const int nch = std::max(1, (M + kPlanChunk - 1) / kPlanChunk);
    // hist[B][nch] | off[B][nch] | tot[B] | counts[2]
    if (ensure(ctx->smeta, sizeof(int4) * std::max(M, 1)) ||
        ensure(ctx->plan_hist, sizeof(int) * (2 * (size_t)nch * kPlanBuckets + kPlanBuckets + 2)))
        return DASH_E_CUDA;
    int *hist = (int *)ctx->plan_hist.p;
    int *off = hist + (size_t)nch * kPlanBuckets;
    int *tot = off + (size_t)nch * kPlanBuckets;
    int *counts = tot + kPlanBuckets;
    PhaseScope ps(ctx, st, PH_ROWSLICE);
    // first kernel of the update: a normal launch (fully ordered after the previous update)
    k_plan_count<<<nch, kPlanChunk, 0, st>>>(b->row_ptr, M, hist, tflag, ctx->tgen);
    ctx->last_launches += 2;  // three kernels under one phase
    return launch_k(true, k_plan_scan, kPlanBuckets, kScanThreads, 0, st, (const int *)hist, nch, off, tot) ||
           launch_k(true, k_plan_scatter, (nch + 3) / 4, 128, 0, st, (const int64_t *)b->row_ptr, b->state_row,
                    b->is_new, M, nch, (const int *)off, (const int *)tot, (int4 *)ctx->smeta.p, counts);
}

const int *plan_counts_of(dash_ctx *ctx, int M) {
    const int nch = std::max(1, (M + kPlanChunk - 1) / kPlanChunk);
    return (const int *)ctx->plan_hist.p + 2 * (size_t)nch * kPlanBuckets + kPlanBuckets;
}

template <int NB>
int run_slicesw(dash_ctx *ctx, cudaStream_t st, SwParams q) {
    using Cf = swk::Cfg<NB>;
    const int grid = ctx->num_sms;
    if (ensure(ctx->sw_scr, sizeof(double) * (size_t)grid * (Cf::NW * Cf::scr_doubles + Cf::NT * 64))) return DASH_E_CUDA;
    q.scratch = (double *)ctx->sw_scr.p;
    q.vtv_tiles = q.scratch + (size_t)grid * Cf::NW * Cf::scr_doubles;
    ensure_smem_attr(k_slicesw<NB>, Cf::smem_bytes());
    k_slicesw<NB><<<grid, Cf::NW * 32, Cf::smem_bytes(), st>>>(q);
    return cudaGetLastError() == cudaSuccess ? 0 : DASH_E_CUDA;
}

int launch_slicesw(dash_ctx *ctx, cudaStream_t st, int RB, int M, const SliceParams &sp) {
    SwParams q{reinterpret_cast<const int32_t *>(sp.items), M, sp.row_ptr, sp.state_row, sp.is_new, sp.XV, sp.U,
               sp.W, sp.C, sp.D, sp.vtv, nullptr, nullptr, sp.err, sp.fallbacks, sp.R, sp.lam, sp.eps, sp.pass,
               sp.final_pass};
    PhaseScope ps(ctx, st, PH_SLICES);
    return RB <= 32 ? run_slicesw<4>(ctx, st, q) : run_slicesw<8>(ctx, st, q);
}

int launch_plan(dash_ctx *ctx, cudaStream_t st, int RB, const SlicePlan &pl, SliceParams sp, int M,
                bool skip_big = false) {
    if (pl.wide) return launch_slicesw(ctx, st, RB, M, sp);
    if (!pl.split) return dispatch_slices(ctx, st, RB, (int)pl.items.size(), sp);
    const int4 *meta = (const int4 *)ctx->smeta.p;
    const int *counts = plan_counts_of(ctx, M);
    {
        PhaseScope ps(ctx, st, PH_SLICES);
        int rc = RB == 4 ? launch_slices3<4>(st, pl.g3, sp, meta, counts)
                 : RB == 8 ? launch_slices3<8>(st, pl.g3, sp, meta, counts)
                           : launch_slices3<16>(st, pl.g3, sp, meta, counts);
        if (rc) return rc;
    }
    SliceParams sb = sp;
    sb.G_slots = sp.G_slots + (int64_t)pl.g3 * sp.R * sp.R;
    if (pl.big_dev) {
        if (pl.gbig == 0 || skip_big) return 0;
        PhaseScope ps(ctx, st, PH_BIG);
        return launch_big(st, pl.gbig, sb, meta, counts);  // DMMA big-slice kernel, plan order
    }
    if (pl.nbig > 0) {
        PhaseScope ps(ctx, st, PH_BIG);
        switch (RB) {
            case 4: return launch_slices2<4>(st, pl.nbig, sb);
            case 8: return launch_slices2<8>(st, pl.nbig, sb);
            default: return launch_slices2<16>(st, pl.nbig, sb);
        }
    }
    return 0;
}

template <int RP, class B>
void launch_xv_t(dash_ctx *ctx, cudaStream_t st, const B *b, int J, const double *V, int R, double *XV) {
    int64_t ntiles = (b->N + 63) / 64;
    int grid = (int)std::min<int64_t>(ntiles, (int64_t)ctx->num_sms * 8);
    if (grid < 1) grid = 1;
    PhaseScope ps(ctx, st, PH_XV);
    k_xv<RP><<<grid, 256, 0, st>>>(b->X, b->ldx, b->N, J, V, R, XV);
}

template <class B>
void launch_xv(dash_ctx *ctx, cudaStream_t st, const B *b, int J, const double *V, int R, double *XV) {
    switch (rank_bucket(R) < 8 ? 8 : rank_bucket(R)) {
        case 8: launch_xv_t<8>(ctx, st, b, J, V, R, XV); break;
        case 16: launch_xv_t<16>(ctx, st, b, J, V, R, XV); break;
        case 32: launch_xv_t<32>(ctx, st, b, J, V, R, XV); break;
        default: launch_xv_t<64>(ctx, st, b, J, V, R, XV); break;
    }
}

template <int RP, class B>
void launch_fgemm_t(dash_ctx *ctx, cudaStream_t st, const B *b, int J, const double *U,
                    const int32_t *row_slice, const double *W, int R, int64_t rps, int nsplit, double *F_slots,
                    double *G_slots) {
    dim3 grid((J + 63) / 64 + (G_slots ? 1 : 0), nsplit);
    PhaseScope ps(ctx, st, PH_FGEMM);
    k_fgemm<RP><<<grid, 256, 0, st>>>(b->X, b->ldx, b->N, J, U, row_slice, b->state_row, W, R, rps, F_slots,
                                      G_slots);
}

template <class B>
void launch_fgemm(dash_ctx *ctx, cudaStream_t st, const B *b, int J, const double *U,
                  const int32_t *row_slice, const double *W, int R, int64_t rps, int nsplit, double *F_slots,
                  double *G_slots = nullptr) {
    switch (rank_bucket(R) < 8 ? 8 : rank_bucket(R)) {
        case 8: launch_fgemm_t<8>(ctx, st, b, J, U, row_slice, W, R, rps, nsplit, F_slots, G_slots); break;
        case 16: launch_fgemm_t<16>(ctx, st, b, J, U, row_slice, W, R, rps, nsplit, F_slots, G_slots); break;
        case 32: launch_fgemm_t<32>(ctx, st, b, J, U, row_slice, W, R, rps, nsplit, F_slots, G_slots); break;
        default: launch_fgemm_t<64>(ctx, st, b, J, U, row_slice, W, R, rps, nsplit, F_slots, G_slots); break;
    }
}

// ---------------------------------------------------------------------------
// k_vsolvew<NB>: the V solve for R in (16, 64] on DMMA tiles.  F = lam F0 + f,
// G = sym(lam G0 + g), V = ridge_solve(G, F^T)^T (stream.py:344-346,
// linalg.py:25-45).  Every CTA factors G + shift I once (one warp: the blocked
// tile Cholesky of dash_slicesw.cuh), then its 8 warps each take 8-row chunks
// of F and solve them against the factor (blocked substitution on DMMA) --
// ~25 us where the one-pivot-at-a-time sweep of k_vsolve_cta<64> takes ~100 us
// (64 block-wide barriers).  A non-SPD / non-finite G leaves the update to the
// reference's fallback chain: the kernel then only marks the launch (flag = its
// generation) and the sweep / LU kernel, launched behind it, runs for real.
// ---------------------------------------------------------------------------
template <int NB>
__global__ void __launch_bounds__(256) k_vsolvew(const double *__restrict__ fg, const double *__restrict__ F_snap,
                                                 const double *__restrict__ G_snap, double lam, int J, int R, double eps,
                                                 double *__restrict__ F, double *__restrict__ G, double *__restrict__ V,
                                                 unsigned long long *err, unsigned int *flag, unsigned int gen) {
    using namespace swk;
    constexpr int NT = NB * (NB + 1) / 2, NWV = 8;
    extern __shared__ __align__(16) double sm[];
    double *Lt = sm, *Li = Lt + 64 * NT;
    const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
    double *Uc = Li + 64 * NB + w * (NB + 1) * 64, *Cs = Uc + 64 * NB;
    __shared__ int okf;
    __shared__ double shv;
    pdl_wait();     // fg from the slot sums
    pdl_trigger();
    const int64_t JR = (int64_t)J * R;
    const double *g = fg + JR;
    for (int e = tid; e < NT * 64; e += 256) {
        const int t = e >> 6, k = e & 63, r = k >> 3, c = (k & 7) ^ ((r & 2) << 1);
        int ib = 0;
        while (tri(ib + 1, 0) <= t) ++ib;
        const int kb = t - tri(ib, 0);
        const int row = 8 * ib + r, col = 8 * kb + c;
        double v = (row == col) ? 1.0 : 0.0;
        if (row < R && col < R) {
            const double m1 = lam * G_snap[row * R + col] + g[row * R + col];
            const double m2 = lam * G_snap[col * R + row] + g[col * R + row];
            v = (m1 + m2) / 2.0;
            if (blockIdx.x == 0) {
                G[row * R + col] = v;
                G[col * R + row] = v;
            }
        }
        Lt[e] = v;
    }
    __syncthreads();
    if (w == 0) {
        double tr = 0.0;
        for (int r = lane; r < R; r += 32) tr += Lt[64 * tri(r >> 3, r >> 3) + toff(r & 7, r & 7)];
        tr = warp_sum(tr);
        if (lane == 0) shv = eps * (tr / R);
    }
    __syncthreads();
    if (tid < R) Lt[64 * tri(tid >> 3, tid >> 3) + toff(tid & 7, tid & 7)] += shv;
    __syncthreads();
    const LaneOff o = lane_offsets();
    if (w == 0) {
        const bool ok = chol_tiles<NB>(Lt, Li, o);
        if (lane == 0) okf = ok ? 1 : 0;
    }
    __syncthreads();
    if (!okf) {  // not SPD: the sweep / LU kernel behind this one takes over (it rewrites F, G, V)
        if (tid == 0) *flag = gen;
        return;
    }
    const int nchunks = (J + 7) / 8;
    for (int ch = blockIdx.x * NWV + w; ch < nchunks; ch += gridDim.x * NWV) {
        const int j = 8 * ch + o.g;
        double x[NB][2];
#pragma unroll
        for (int jb = 0; jb < NB; ++jb)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int col = 8 * jb + o.c0 + e;
                double f = 0.0;
                if (j < J && col < R) {
                    f = lam * F_snap[(int64_t)j * R + col] + fg[(int64_t)j * R + col];
                    F[(int64_t)j * R + col] = f;
                }
                x[jb][e] = f;
            }
        __syncwarp();
        solve_chunk<NB>(x, Lt, Li, Uc, Cs, o);
        bool fin = true;
#pragma unroll
        for (int jb = 0; jb < NB; ++jb)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int col = 8 * jb + o.c0 + e;
                if (j < J && col < R) {
                    V[(int64_t)j * R + col] = x[jb][e];
                    fin = fin && finite_d(x[jb][e]);
                }
            }
        if (!fin) report_error(err, -1, DASH_E_NONFINITE);
        __syncwarp();
    }
}

// returns true if k_vsolvew was launched (the caller then launches the fallback kernel gated on the flag)
template <int NB>
bool launch_vsolvew(dash_ctx *ctx, cudaStream_t st, const double *fg, double lam, int J, int R, double eps, double *F,
                    double *G, double *V, unsigned int &gen) {
    static const bool off = getenv("DASH_OLD_VSOLVE") != nullptr;  // A/B switch: the sweep kernels only
    if (off) return false;
    constexpr int NT = NB * (NB + 1) / 2;
    const size_t smem = sizeof(double) * 64 * (NT + NB + 8 * (NB + 1));
    ensure_smem_attr(k_vsolvew<NB>, smem);
    gen = ++ctx->vs_gen;
    if (gen == 0) gen = ++ctx->vs_gen;  // 0 is the flag's resting value
    const int blocks = std::max(1, ((J + 7) / 8 + 7) / 8);
    ctx->last_launches++;
    return launch_k(pdl_site("vsw"), k_vsolvew<NB>, blocks, 256, smem, st, fg, (const double *)ctx->fsnap.p,
                    (const double *)ctx->gsnap.p, lam, J, R, eps, F, G, V, ctx->err, ctx->vs_flag, gen) == 0;
}

template <int RB>
void launch_vsolve_t(dash_ctx *ctx, cudaStream_t st, const double *fg, double lam, int J, int R, double eps,
                     double *F, double *G, double *V) {
    PhaseScope ps(ctx, st, PH_VSOLVE);
    static const bool old_vsolve = getenv("DASH_CHOL_VSOLVE") != nullptr;  // A/B: per-warp Cholesky variant
    if constexpr (RB <= 16) {
        if (!old_vsolve) {
            launch_k(pdl_site("vs"), k_vsolve2<RB>, (J + 127) / 128, 128, 0, st, fg, (const double *)ctx->fsnap.p,
                     (const double *)ctx->gsnap.p, lam, J, R, eps, F, G, V, ctx->err, ctx->fallbacks);
            return;
        }
    }
    constexpr int NWV = RB <= 16 ? 4 : 1;
    int blocks = (J + NWV * 32 - 1) / (NWV * 32);
    const unsigned int *only_if = nullptr;
    unsigned int gen = 0;
    if constexpr (RB == 32) {
        if (launch_vsolvew<4>(ctx, st, fg, lam, J, R, eps, F, G, V, gen)) only_if = ctx->vs_flag;
    }
    launch_k(true, k_vsolve<RB, NWV>, blocks, NWV * 32, 0, st, fg, (const double *)ctx->fsnap.p,
             (const double *)ctx->gsnap.p, lam, J, R, eps, F, G, V, ctx->err, ctx->fallbacks, only_if, gen);
}

// out[0:width] = column sums of slots (nslots x width), deterministic order
int colsum(dash_ctx *ctx, cudaStream_t st, const double *slots, int nslots, int64_t width, double *out) {
    const int nseg = std::max(1, (nslots + kSeg - 1) / kSeg);
    if (ensure(ctx->part, sizeof(double) * nseg * width)) return DASH_E_CUDA;
    double *part = (double *)ctx->part.p;
    const int bx = (int)((width + 127) / 128);
    if (nslots == 0) {
        cudaMemsetAsync(out, 0, sizeof(double) * width, st);
        return 0;
    }
    k_colsum_part<<<dim3(bx, nseg), 128, 0, st>>>(slots, nslots, width, part);
    k_colsum_final<<<bx, 128, 0, st>>>(part, nseg, width, out);
    return 0;
}

// column sums of two slot arrays (F slots and G slots) in two launches
int colsum2(dash_ctx *ctx, cudaStream_t st, const double *sa, int na, int64_t wa, double *oa, const double *sb,
            int nb, int64_t wb, double *ob) {
    if (na == 0 || nb == 0) return colsum(ctx, st, sa, na, wa, oa) || colsum(ctx, st, sb, nb, wb, ob);
    ColSumJob a{sa, nullptr, oa, wa, na, std::max(1, (na + kSeg - 1) / kSeg), (int)((wa + 127) / 128)};
    ColSumJob b{sb, nullptr, ob, wb, nb, std::max(1, (nb + kSeg - 1) / kSeg), (int)((wb + 127) / 128)};
    if (ensure(ctx->part, sizeof(double) * (a.nseg * wa + b.nseg * wb))) return DASH_E_CUDA;
    a.part = (double *)ctx->part.p;
    b.part = a.part + a.nseg * wa;
    ctx->last_launches++;  // two kernels under one phase
    return launch_k(pdl_site("cs1"), k_colsum_part2, a.bx * a.nseg + b.bx * b.nseg, 128, 0, st, a, b) ||
           launch_k(pdl_site("cs2"), k_colsum_final2, a.bx + b.bx, 128, 0, st, a, b);
}

// ---- streaming (TMA ring) GEMM path: J, ldx, R even; ring fits in shared memory
template <int RP>
bool stream_ok_t(int J, int64_t ldx, int R) {
    if ((J & 1) || (ldx & 1) || (R & 1)) return false;
    const int JP = ((J + 7) / 8) * 8;
    if ((JP / 8) * (RP / 8) > 64) return false;
    const size_t lim = 220 * 1024;
    return StreamSmem<RP>::xv_bytes(J) <= lim && StreamSmem<RP>::f_bytes(J) <= lim;
}
bool stream_ok(int J, int64_t ldx, int R) {
    const int RB = rank_bucket(R);
    if (RB > 16) return false;  // US is produced by k_slices2 (R <= 16)
    return RB <= 8 ? stream_ok_t<8>(J, ldx, R) : stream_ok_t<16>(J, ldx, R);
}

// ---- tensor-map path (R bucket 16): box 16 doubles x 32 rows, 128B swizzle, OOB rows zero-filled
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {  // thread-safe one-time init
        cudaDriverEntryPointQueryResult q;
        void *f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
        cudaGetLastError();
        return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    }();
    return fn;
}

bool make_box_map(CUtensorMap *map, const double *base, int64_t cols, int64_t rows, int64_t ld,
                  int box_rows = kTR) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
    cuuint32_t box[2] = {16, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_box_map(CUtensorMap *map, const float *base, int64_t cols, int64_t rows, int64_t ld) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(float)};
    cuuint32_t box[2] = {32, (cuuint32_t)kTR};
    cuuint32_t es[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool tma_ok(const dash_batch_f32 *b, int J, int R) {
    const size_t lim = 220 * 1024;
    return rank_bucket(R) == 16 && !(R & 1) && !(b->ldx & 3) && (reinterpret_cast<uintptr_t>(b->X) & 15) == 0 &&
           b->N < (int64_t)1 << 31 && TmaSmem32::strips(J) <= 8 && TmaSmem32::xv_bytes(J) <= lim &&
           TmaSmem32::f_bytes(J) <= lim && encode_fn() != nullptr;
}

int launch_xv3(dash_ctx *ctx, cudaStream_t st, const dash_batch_f32 *b, int J, const double *V, int R, double *XV,
               const FusedPrologue &pro, bool pdl, const uint32_t *tflag = nullptr) {
    CUtensorMap mx;
    if (!make_box_map(&mx, b->X, J, b->N, b->ldx)) return DASH_E_CUDA;
    const size_t smem = TmaSmem32::xv_bytes(J);
    ensure_smem_attr(k_xv3f, smem);
    PhaseScope ps(ctx, st, PH_XV);
    return launch_k(pdl && pdl_site("xv3f"), k_xv3f, ctx->num_sms, kCW * 32 + 32, smem, st, mx, b->N, J, V, R, XV, pro,
                    tflag, ctx->tgen);
}

int launch_f3(dash_ctx *ctx, cudaStream_t st, const dash_batch_f32 *b, int J, const double *US, int R,
              double *F_slots, const uint32_t *tflag = nullptr) {
    CUtensorMap mx, mu;
    if (!make_box_map(&mx, b->X, J, b->N, b->ldx) || !make_box_map(&mu, US, R, b->N, R)) return DASH_E_CUDA;
    const size_t smem = TmaSmem32::f_bytes(J);
    ensure_smem_attr(k_fgemm3f, smem);
    PhaseScope ps(ctx, st, PH_FGEMM);
    return launch_k(pdl_site("f3f"), k_fgemm3f, ctx->num_sms, kCW * 32 + 32, smem, st, mx, mu, b->N, J, R, F_slots,
                    tflag, ctx->tgen);
}

// U_new of the FP32 data mode: FP64 working copy -> caller's FP32 array
__global__ void k_u_to_f32(const double *__restrict__ U, int64_t n, float *__restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (float)U[i];
}

bool tma_ok(const dash_batch_f64 *b, int J, int R) {
    const size_t lim = 220 * 1024;
    return rank_bucket(R) == 16 && !(R & 1) && !(b->ldx & 1) && (reinterpret_cast<uintptr_t>(b->X) & 15) == 0 &&
           b->N < (int64_t)1 << 31 && TmaSmem::strips(J) <= 16 && TmaSmem::xv_bytes(J) <= lim &&
           TmaSmem::f_bytes(J) <= lim && encode_fn() != nullptr;
}

int launch_xv3(dash_ctx *ctx, cudaStream_t st, const dash_batch_f64 *b, int J, const double *V, int R, double *XV,
               const FusedPrologue &pro, bool pdl, const uint32_t *tflag = nullptr) {
    CUtensorMap mx;
    if (!make_box_map(&mx, b->X, J, b->N, b->ldx)) return DASH_E_CUDA;
    const size_t smem = TmaSmem::xv_bytes(J);
    ensure_smem_attr(k_xv3, smem);
    PhaseScope ps(ctx, st, PH_XV);
    return launch_k(pdl, k_xv3, ctx->num_sms, kCW * 32 + 32, smem, st, mx, b->N, J, V, R, XV, pro, tflag, ctx->tgen);
}

template <int MAXS>
void launch_f3_t(dash_ctx *ctx, cudaStream_t st, const CUtensorMap &mx, const CUtensorMap &mu, int64_t N, int J,
                 int R, double *F_slots, const uint32_t *tflag, double *G_slots) {
    const size_t smem = TmaSmem::f_bytes(J);
    ensure_smem_attr(k_fgemm3<MAXS>, smem);
    PhaseScope ps(ctx, st, PH_FGEMM);
    launch_k(pdl_site("f3"), k_fgemm3<MAXS>, ctx->num_sms, kCW * 32 + 32, smem, st, mx, mu, N, J, R, F_slots, tflag,
             ctx->tgen, G_slots);
}

// F slots (and, with G_slots, the G slots of sum US^T US) over the tiles marked in tflag
int launch_f3(dash_ctx *ctx, cudaStream_t st, const dash_batch_f64 *b, int J, const double *US, int R,
              double *F_slots, const uint32_t *tflag = nullptr, double *G_slots = nullptr) {
    CUtensorMap mx, mu;
    if (!make_box_map(&mx, b->X, J, b->N, b->ldx) || !make_box_map(&mu, US, R, b->N, R)) return DASH_E_CUDA;
    if (TmaSmem::strips(J) <= kCW) launch_f3_t<1>(ctx, st, mx, mu, b->N, J, R, F_slots, tflag, G_slots);
    else launch_f3_t<2>(ctx, st, mx, mu, b->N, J, R, F_slots, tflag, G_slots);
    return 0;
}

// fused big-slice chain (dash_bigx.cuh): pre (A systems, toff), the streaming kernel, post
template <class B>
int launch_bigx(dash_ctx *ctx, cudaStream_t st, const B *b, const BigxParams &bp) {
    using TX = typename std::remove_const<typename std::remove_pointer<decltype(b->X)>::type>::type;
    using SM = BigxSmemT<TX>;
    if (bp.T == 0) return 0;
    const int nbig = ctx->bigx_nbig;
    PhaseScope ps(ctx, st, PH_BIG);
    ctx->last_launches += 1;  // two kernels under one phase (pre, streaming); post after the F GEMM
    if (launch_k(pdl_site("bxpre"), k_bigx_pre, 1 + (nbig + 7) / 8, 256, 0, st, bp)) return DASH_E_CUDA;
    CUtensorMap mx;
    if (!make_box_map(&mx, b->X, bp.J, b->N, b->ldx)) return DASH_E_CUDA;
    const size_t smem = SM::bytes(bp.J);
    const int js = SM::strips(bp.J);
    auto go = [&](auto kern) {
        ensure_smem_attr(kern, smem);
        return launch_k(pdl_site("bigx"), kern, bp.G, kBxThreads, smem, st, mx, bp);
    };
    int rc;
    // J <= 128 (the fused path's limit): <= 8 FP64 / 4 FP32 strips over kBxB X^T U warps
    constexpr int MS = kBxB >= 8 ? 1 : 2;  // P strips per X^T U warp for up to 8 strips
    if constexpr (SM::F32)  // float boxes: 32 columns per strip (<= 4)
        rc = js == 4 ? go(k_bigx<1, 4, float>) : go(k_bigx<1, 0, float>);
    else
        rc = js == 8 ? go(k_bigx<MS, 8, double>) : js <= kBxB ? go(k_bigx<1, 0, double>) : go(k_bigx<MS, 0, double>);
    return rc;
}

int launch_bigx_post(dash_ctx *ctx, cudaStream_t st, const BigxParams &bp) {
    if (bp.T == 0) return 0;
    PhaseScope ps(ctx, st, PH_BIGPOST);
    return launch_k(pdl_site("bxpost"), k_bigx_post, ctx->bigx_nbig, 256, 0, st, bp);
}

// ---- wide-J tensor-map GEMMs (dash_widej.cuh)
bool widej_ok(const dash_batch_f64 *b, int J, int R, const double *V) {
    static const bool off = getenv("DASH_NO_WIDEJ") != nullptr;  // A/B switch: the generic register-staged GEMMs
    return !off && J > 128 && !(R & 1) && R <= 64 && !(b->ldx & 1) && (reinterpret_cast<uintptr_t>(b->X) & 15) == 0 &&
           (reinterpret_cast<uintptr_t>(V) & 15) == 0 && b->N < ((int64_t)1 << 31) - 64 && encode_fn() != nullptr;
}

template <int RP>
int launch_xvw_t(dash_ctx *ctx, cudaStream_t st, const CUtensorMap &mx, const CUtensorMap &mv, int64_t N, int J, int R,
                 double *XV) {
    constexpr size_t smem = WideCfg<RP>::xv_bytes();
    ensure_smem_attr(k_xvw<RP>, smem);
    const int grid = (int)std::min<int64_t>(ctx->num_sms, (N + 63) / 64);
    k_xvw<RP><<<grid, kCW * 32 + 32, smem, st>>>(mx, mv, N, J, R, XV);
    return cudaGetLastError() == cudaSuccess ? 0 : DASH_E_CUDA;
}

int launch_xvw(dash_ctx *ctx, cudaStream_t st, const dash_batch_f64 *b, int J, const double *V, int R, double *XV) {
    CUtensorMap mx, mv;
    if (!make_box_map(&mx, b->X, J, b->N, b->ldx) || !make_box_map(&mv, V, R, J, R, 64)) return DASH_E_CUDA;
    PhaseScope ps(ctx, st, PH_XV);
    const int RB = rank_bucket(R);
    return RB <= 16 ? launch_xvw_t<16>(ctx, st, mx, mv, b->N, J, R, XV)
           : RB <= 32 ? launch_xvw_t<32>(ctx, st, mx, mv, b->N, J, R, XV)
                      : launch_xvw_t<64>(ctx, st, mx, mv, b->N, J, R, XV);
}

template <int RP>
int launch_fw_t(dash_ctx *ctx, cudaStream_t st, const CUtensorMap &mx, const CUtensorMap &mu, int64_t N, int J, int R,
                double *F_slots, double *G_slots) {
    constexpr size_t smem = WideCfg<RP>::f_bytes();
    ensure_smem_attr(k_fgemmw<RP>, smem);
    k_fgemmw<RP><<<(unsigned)(ctx->wnj * ctx->nsplit), kCW * 32 + 32, smem, st>>>(mx, mu, N, J, R, ctx->rps, ctx->wnj,
                                                                                 F_slots, G_slots);
    return cudaGetLastError() == cudaSuccess ? 0 : DASH_E_CUDA;
}

int launch_fw(dash_ctx *ctx, cudaStream_t st, const dash_batch_f64 *b, int J, const double *US, int R, double *F_slots,
              double *G_slots) {
    CUtensorMap mx, mu;
    if (!make_box_map(&mx, b->X, J, b->N, b->ldx) || !make_box_map(&mu, US, R, b->N, R)) return DASH_E_CUDA;
    PhaseScope ps(ctx, st, PH_FGEMM);
    const int RB = rank_bucket(R);
    return RB <= 16 ? launch_fw_t<16>(ctx, st, mx, mu, b->N, J, R, F_slots, G_slots)
           : RB <= 32 ? launch_fw_t<32>(ctx, st, mx, mu, b->N, J, R, F_slots, G_slots)
                      : launch_fw_t<64>(ctx, st, mx, mu, b->N, J, R, F_slots, G_slots);
}
int launch_xvw(dash_ctx *, cudaStream_t, const dash_batch_f32 *, int, const double *, int, double *) { return DASH_E_ARG; }
int launch_fw(dash_ctx *, cudaStream_t, const dash_batch_f32 *, int, const double *, int, double *, double *) {
    return DASH_E_ARG;
}

template <int RP>
void launch_xv2_t(dash_ctx *ctx, cudaStream_t st, const dash_batch_f64 *b, int J, const double *V, int R, double *XV) {
    const size_t smem = StreamSmem<RP>::xv_bytes(J);
    ensure_smem_attr(k_xv2<RP>, smem);
    PhaseScope ps(ctx, st, PH_XV);
    k_xv2<RP><<<ctx->num_sms, kCW * 32 + 32, smem, st>>>(b->X, b->ldx, b->N, J, V, R, XV);
}

template <int RP, int MAXT>
void launch_f2_tt(dash_ctx *ctx, cudaStream_t st, const dash_batch_f64 *b, int J, const double *US, int R,
                  double *F_slots) {
    const size_t smem = StreamSmem<RP>::f_bytes(J);
    ensure_smem_attr(k_fgemm2<RP, MAXT>, smem);
    PhaseScope ps(ctx, st, PH_FGEMM);
    k_fgemm2<RP, MAXT><<<ctx->num_sms, kCW * 32 + 32, smem, st>>>(b->X, b->ldx, b->N, J, US, R, F_slots);
}

template <int RP>
void launch_f2_t(dash_ctx *ctx, cudaStream_t st, const dash_batch_f64 *b, int J, const double *US, int R,
                 double *F_slots) {
    const int need = ((((J + 7) / 8) * (RP / 8)) + 7) / 8;
    if (need <= 1) launch_f2_tt<RP, 1>(ctx, st, b, J, US, R, F_slots);
    else if (need <= 2) launch_f2_tt<RP, 2>(ctx, st, b, J, US, R, F_slots);
    else if (need <= 4) launch_f2_tt<RP, 4>(ctx, st, b, J, US, R, F_slots);
    else launch_f2_tt<RP, 8>(ctx, st, b, J, US, R, F_slots);
}

bool valid_state(const dash_state_f64 *s) {
    return s && s->R >= 1 && s->R <= DASH_MAX_RANK && s->J >= 1 && s->passes >= 1 && s->forgetting > 0.0 &&
           s->forgetting <= 1.0;
}

}  // namespace

// One pass of the update (U / c / D / W for the batch's slices, F and G fresh
// sums into fg_out).  B = dash_batch_f64 or dash_batch_f32 (the FP32 data
// mode: X and U_out in FP32; the slice kernels then write an FP64 working U
// that is rounded into U_out after the final pass).
template <class B, typename TU>
int pass_begin_impl(dash_ctx *ctx, void *stream, const B *b, dash_state_f64 *s, TU *U_out, double *v_used_out,
                    double eps, int32_t pass, double *fg_out) {
    constexpr bool f32 = std::is_same<B, dash_batch_f32>::value;
    static_assert(std::is_same<TU, typename std::conditional<f32, float, double>::type>::value, "U type");
    if (!ctx || !b || !valid_state(s) || !U_out || !v_used_out || !fg_out) return DASH_E_ARG;
    if (b->M < 0 || b->N < 0 || b->N > DASH_MAX_BATCH_ROWS || (b->N > 0 && b->ldx < s->J) || pass < 0 ||
        pass >= s->passes)
        return DASH_E_ARG;
    const int J = s->J, R = s->R;
    cudaStream_t st = (cudaStream_t)stream;
    const int RB = rank_bucket(R);
    const int64_t N = b->N;
    const int M = b->M;
    const int last = pass == s->passes - 1;
    static const bool host_timing = getenv("DASH_HOST_TIMING") != nullptr;
    auto tnow = [] { return std::chrono::steady_clock::now(); };
    auto t0 = tnow();
    ctx->cur_pass = pass;
    cudaStream_t pst = st;  // stream of the plan kernels (the staging side stream when the plan runs ahead)
    if (pass == 0) {
        ctx->side_plan = false;
        ctx->last_launches = 0;
        if (!ctx->plan_p) ctx->plan_p = new SlicePlan();
        plan_of(ctx) = make_plan(b->row_ptr_host, M, RB, R, ctx->num_sms);
        if (host_timing) fprintf(stderr, "[dash host] plan %.1f us\n", std::chrono::duration<double, std::micro>(tnow() - t0).count());
        ctx->nitems = plan_of(ctx).nslots;
        const std::vector<int4> &items = plan_of(ctx).items;
        if constexpr (f32) {  // FP32 X: tensor-map path, else the generic GEMMs (no row-copy ring)
            ctx->tma = N > 0 && tma_ok(b, J, R);
            ctx->stream = ctx->tma;
        } else {
            ctx->stream = stream_ok(J, b->ldx, R) && N > 0;
        }
        plan_fsplit(ctx, N, J, ctx->nsplit, ctx->rps);
        if (ctx->stream) ctx->nsplit = ctx->num_sms * (f32 ? TmaSmem32::row_groups(J) : 1);
        ctx->wtma = false;
        if constexpr (!f32) {
            if (!ctx->stream && N > 0 && widej_ok(b, J, R, s->V)) {
                // column blocks x row ranges (multiples of 32 rows), about one CTA per SM
                const int fc = RB <= 32 ? WideCfg<32>::FC : WideCfg<64>::FC;
                ctx->wnj = (J + fc - 1) / fc;
                // k_slicesw's G term rides on the F GEMM: 2 tiles per warp must cover the (RB/8)^2 tiles
                ctx->wtma = !plan_of(ctx).wide || (RB / 8) * (RB / 8) <= 16 * ctx->wnj;
            }
            if (ctx->wtma) {
                const int64_t nrow = std::max<int64_t>(1, ctx->num_sms / ctx->wnj);
                ctx->rps = std::max<int64_t>(32, ((N + nrow - 1) / nrow + 31) / 32 * 32);
                ctx->nsplit = (N + ctx->rps - 1) / ctx->rps;
            }
        }
        ctx->swide = plan_of(ctx).wide;
        if (ctx->swide) ctx->nitems = (int)ctx->nsplit;  // G slots: one per F-GEMM row split
        if constexpr (!f32) ctx->tma = ctx->stream && tma_ok(b, J, R);
        {
            static const bool no_bigx = getenv("DASH_NO_BIGX") != nullptr;  // A/B switch: the k_big path
            const SlicePlan &pl = plan_of(ctx);
            ctx->bigx = !no_bigx && ctx->tma && pl.big_dev && pl.gbig > 0 && J * 16 <= kPostPer * 256 &&
                        BigxSmemT<typename std::conditional<f32, float, double>::type>::bytes(J) <= 227 * 1024;
            // fused small-slice kernel: same eligibility as the fused big path (FP64, R
            // bucket 16 and even, J <= 128, tensor-map X); big slices then need k_bigx
            // opt-in (DASH_SMALLX=1): measured slower than k_xv3 -> k_slices3 -> k_fgemm3 on the
            // large config (0.72 vs 0.58 ms / update; latency-bound solver warps and an
            // instruction footprint beyond the 32 KB L1.5 I-cache)
            static const bool use_smallx = getenv("DASH_SMALLX") != nullptr;
            ctx->smallx = !f32 && use_smallx && !no_bigx && ctx->tma && pl.big_dev && J <= 128 &&
                          (ctx->bigx || pl.gbig == 0);
            ctx->sx_grid = ctx->smallx ? ctx->num_sms : 0;
            if (ctx->smallx) {
                const int nch = std::max(1, (M + kSxChunk - 1) / kSxChunk);
                if (ensure(ctx->sx_tmp, sizeof(int4) * (size_t)nch * kSxChunk) ||
                    ensure(ctx->sx_units, sizeof(int) * kSxRec * (size_t)std::max(M, 1))) return DASH_E_CUDA;
                if (ctx->sx_meta.cap < sizeof(int) * (2 * (size_t)nch + 8)) {
                    if (ensure(ctx->sx_meta, sizeof(int) * (2 * (size_t)nch + 8))) return DASH_E_CUDA;
                    cudaMemsetAsync(ctx->sx_meta.p, 0, ctx->sx_meta.cap, st);  // done counter starts at 0
                }
            }
            ctx->bigx_nbig = ctx->bigx ? pl.gbig : 0;
            ctx->bigx_grid = ctx->bigx ? (int)std::min<int64_t>(ctx->num_sms, pl.big_tiles) : 0;
            if (ctx->smallx) ctx->nitems = ctx->sx_grid + pl.gbig;  // G slots: one per small-kernel CTA + big slice
            {
                // side-stream plan: only for batches staged by dash_stage_meta (their index arrays were
                // copied on meta_stream, so the plan kernels there are ordered behind the copy)
                static const bool side_off = getenv("DASH_NO_SIDE_PLAN") != nullptr;
                // (small updates are host-bound: the three extra stream calls would cost more than they hide)
                const bool will_plan = pl.split && M > 0 && N >= 32768 && !ctx->smallx;
                ctx->side_plan = will_plan && !side_off && !ctx->prof && ctx->meta_stream && ctx->mring_last >= 0 &&
                                 (const void *)b->row_ptr == (const void *)ctx->mring[ctx->mring_last].dev;
                if (ctx->side_plan) {
                    std::swap(ctx->smeta, ctx->pset_alt.smeta);
                    std::swap(ctx->plan_hist, ctx->pset_alt.plan_hist);
                    std::swap(ctx->tflag, ctx->pset_alt.tflag);
                    std::swap(ctx->tgen, ctx->pset_alt.tgen);
                    std::swap(ctx->pset_free, ctx->pset_alt.free_ev);
                    std::swap(ctx->pset_used, ctx->pset_alt.used);
                    pst = ctx->meta_stream;
                    // the update that last read this set must have been issued in full
                    if (ctx->pset_used && cudaStreamWaitEvent(pst, ctx->pset_free, 0) != cudaSuccess) return DASH_E_CUDA;
                }
            }
            if (ctx->bigx) {
                const size_t tb = sizeof(uint32_t) * (size_t)((N + kTR - 1) / kTR + 16);
                if (ctx->tflag.cap < tb) {  // zeroed once: marks are generation-tagged
                    if (ensure(ctx->tflag, tb)) return DASH_E_CUDA;
                    cudaMemsetAsync(ctx->tflag.p, 0, ctx->tflag.cap, pst);
                }
                if (++ctx->tgen == 0) {  // generation wrapped: clear, restart at 1
                    cudaMemsetAsync(ctx->tflag.p, 0, ctx->tflag.cap, pst);
                    ctx->tgen = 1;
                }
            }
            if (ctx->bigx && (ensure(ctx->bx_ms, sizeof(double) * (size_t)pl.gbig * 16 * kBxMP) ||
                              ensure(ctx->bx_toff, sizeof(int) * ((size_t)pl.gbig + 1)) ||
                              ensure(ctx->bx_parts, sizeof(double) * (size_t)(pl.gbig + ctx->bigx_grid) *
                                                        BigxSmem::part_doubles(J))))
                return DASH_E_CUDA;
        }
        if (ensure(ctx->xv, sizeof(double) * std::max<int64_t>(N, 1) * R) ||
            ensure(ctx->row_slice, sizeof(int32_t) * std::max<int64_t>(N, 1)) ||
            ensure(ctx->gslots, sizeof(double) * std::max(ctx->nitems, 1) * R * R) ||
            ensure(ctx->fslots, sizeof(double) * (ctx->nsplit + ctx->bigx_nbig) * J * R) ||
            ensure(ctx->vtv, sizeof(double) * R * R) ||
            ensure(ctx->fsnap, sizeof(double) * J * R) || ensure(ctx->gsnap, sizeof(double) * R * R) ||
            ((ctx->stream || ctx->smallx || ctx->wtma) && ensure(ctx->us, sizeof(double) * std::max<int64_t>(N, 1) * R)) ||
            (f32 && ensure(ctx->u64, sizeof(double) * std::max<int64_t>(N, 1) * R)))
            return DASH_E_CUDA;
        if (!items.empty() && stage_items(ctx, st, items)) return DASH_E_CUDA;
        ctx->planned = plan_of(ctx).split && M > 0 && N > 0 && (!ctx->smallx || ctx->bigx);
        if (ctx->planned &&
            device_plan(ctx, pst, b, ctx->bigx ? (uint32_t *)ctx->tflag.p : nullptr))
            return DASH_E_CUDA;
        if (ctx->side_plan && (cudaEventRecord(ctx->plan_ev, pst) != cudaSuccess ||
                               cudaStreamWaitEvent(st, ctx->plan_ev, 0) != cudaSuccess))
            return DASH_E_CUDA;
        if (M > 0 && !ctx->stream && (!ctx->wtma || ctx->swide)) {  // row -> slice map: the generic F GEMM, k_us_rows
            PhaseScope ps(ctx, st, PH_ROWSLICE);
            k_row_slice<<<std::min(ctx->num_sms * 4, (M + 7) / 8 + 1), 256, 0, st>>>(b->row_ptr, M,
                                                                                    (int32_t *)ctx->row_slice.p);
        }
    }
    double *XV = (double *)ctx->xv.p;
    double *Ud = f32 ? (double *)ctx->u64.p : (double *)(void *)U_out;  // U written by the slice kernels
    double *Fsl = (double *)ctx->fslots.p, *Gsl = (double *)ctx->gslots.p;
    const bool fused_pro = (ctx->tma || ctx->smallx) && N > 0;  // k_xv3 / the small-path planner run the prologue
    if constexpr (!f32) if (ctx->smallx && N > 0) {
        // planner (pass 0) + pass prologue, then the fused small-slice kernel
        const int nch = pass == 0 ? std::max(1, (M + kSxChunk - 1) / kSxChunk) : 0;
        int *sxm = (int *)ctx->sx_meta.p;
        const int nch_all = std::max(1, (M + kSxChunk - 1) / kSxChunk);
        SxPlan pl{b->row_ptr, M, nch, (int4 *)ctx->sx_tmp.p, sxm, sxm + nch_all, (int *)ctx->sx_units.p,
                  sxm + 2 * nch_all + 1, (unsigned int *)(sxm + 2 * nch_all + 2), b->state_row, b->is_new};
        const FusedPrologue pro{(double *)ctx->vtv.p, s->F, s->G, (double *)ctx->fsnap.p, (double *)ctx->gsnap.p,
                                v_used_out, pass == 0, last};
        {
            PhaseScope ps(ctx, st, PH_XV);
            // PDL only behind the plan kernels: otherwise the prologue reads the V / F / G
            // the previous update (or pass) just wrote -> normal launch
            if (launch_k(pass == 0 && ctx->planned && pdl_site("sxwalk"), k_sx_walk, nch + sx_prologue_blocks(R), 256, 0, st, pl, pro, (const double *)s->V,
                         J, R))
                return DASH_E_CUDA;
            if (nch > 0) {
                ctx->last_launches++;
                if (launch_k(pdl_site("sxcopy"), k_sx_copy, nch, 256, 0, st, pl)) return DASH_E_CUDA;
            }
        }
        CUtensorMap m8, m16, m32;
        if (!make_box_map(&m8, b->X, J, b->N, b->ldx, 8) || !make_box_map(&m16, b->X, J, b->N, b->ldx, 16) ||
            !make_box_map(&m32, b->X, J, b->N, b->ldx, 32))
            return DASH_E_CUDA;
        SxParams sp{(const int *)ctx->sx_units.p, sxm + 2 * nch_all + 1, b->row_ptr, b->state_row, b->is_new,
                    s->V, (const double *)ctx->vtv.p, s->W, s->C, s->D, (double *)(void *)U_out,
                    (double *)ctx->us.p, (double *)ctx->fslots.p, (double *)ctx->gslots.p, ctx->err,
                    ctx->fallbacks, J, R, s->forgetting, eps, pass, last, 0};
        static const bool sweep_only = getenv("DASH_S3_SWEEP") != nullptr;
        sp.sweep_only = sweep_only ? 1 : 0;
        {
            PhaseScope ps(ctx, st, PH_SLICES);
            if (launch_smallx(ctx, st, m8, m16, m32, sp, ctx->sx_grid)) return DASH_E_CUDA;
        }
    }
    if (!fused_pro) {
        PhaseScope ps(ctx, st, PH_PROLOGUE);
        const int nvb = (R * R + kVtvWarps - 1) / kVtvWarps;
        k_prologue<<<nvb + std::max(1, std::min(16, (J * R + 255) / 256)), kVtvWarps * 32, 0, st>>>(
            s->V, J, R, (double *)ctx->vtv.p, s->F, s->G, (double *)ctx->fsnap.p,
                                      (double *)ctx->gsnap.p, v_used_out, pass == 0, last, nvb);
    }
    if (N > 0) {
        if (ctx->smallx) {
            // done above
        } else if (ctx->tma) {
            const FusedPrologue pro{(double *)ctx->vtv.p, s->F, s->G, (double *)ctx->fsnap.p, (double *)ctx->gsnap.p,
                                    v_used_out, pass == 0, last};
            // PDL only behind the plan kernels (pass 0); a later pass follows the V solve
            // (not when the plan ran on the side stream: the kernel before this one is then the previous update's)
            if (launch_xv3(ctx, st, b, J, s->V, R, XV, pro, pass == 0 && !ctx->side_plan,
                           ctx->bigx ? (const uint32_t *)ctx->tflag.p : nullptr))
                return DASH_E_CUDA;
        } else if (ctx->stream) {
            if constexpr (!f32) {
                if (rank_bucket(R) <= 8) launch_xv2_t<8>(ctx, st, b, J, s->V, R, XV);
                else launch_xv2_t<16>(ctx, st, b, J, s->V, R, XV);
            }
        } else if (ctx->wtma) {
            if (launch_xvw(ctx, st, b, J, s->V, R, XV)) return DASH_E_CUDA;
        } else {
            launch_xv(ctx, st, b, J, s->V, R, XV);
        }
        SliceParams sp;
        sp.items = (const int4 *)ctx->items.p;
        sp.row_ptr = b->row_ptr;
        sp.state_row = b->state_row;
        sp.is_new = b->is_new;
        sp.XV = XV;
        sp.U = Ud;
        sp.US = (ctx->stream || ctx->wtma) ? (double *)ctx->us.p : nullptr;
        sp.W = s->W;
        sp.C = s->C;
        sp.D = s->D;
        sp.vtv = (const double *)ctx->vtv.p;
        sp.G_slots = Gsl;
        sp.err = ctx->err;
        sp.fallbacks = ctx->fallbacks;
        sp.R = R;
        sp.lam = s->forgetting;
        sp.eps = eps;
        sp.pass = pass;
        sp.final_pass = last;
        if (!ctx->smallx && launch_plan(ctx, st, RB, plan_of(ctx), sp, M, ctx->bigx)) return DASH_E_CUDA;
        if (ctx->wtma && ctx->swide) {  // k_slicesw leaves US to this pass
            PhaseScope ps(ctx, st, PH_SLICES);
            const int64_t n = N * R;
            k_us_rows<<<(int)std::min<int64_t>((n + 255) / 256, (int64_t)ctx->num_sms * 16), 256, 0, st>>>(
                Ud, (const int32_t *)ctx->row_slice.p, b->state_row, s->W, R, n, (double *)ctx->us.p);
        }
        BigxParams bp{};
        {
            if (ctx->bigx) {
                bp.meta = (const int4 *)ctx->smeta.p;
                bp.plan_counts = plan_counts_of(ctx, M);
                bp.V = s->V;
                bp.vtv = (const double *)ctx->vtv.p;
                bp.W = s->W;
                bp.C = s->C;
                bp.Wo = s->W;
                bp.Co = s->C;
                bp.D = s->D;
                bp.U = Ud;
                bp.US = (double *)ctx->us.p;
                bp.ms = (double *)ctx->bx_ms.p;
                bp.toff = (int *)ctx->bx_toff.p;
                bp.parts = (double *)ctx->bx_parts.p;
                bp.F_slots = Fsl + (int64_t)(ctx->smallx ? ctx->sx_grid : ctx->nsplit) * J * R;
                bp.G_slots = Gsl + (int64_t)(ctx->smallx ? ctx->sx_grid : plan_of(ctx).g3) * R * R;
                bp.err = ctx->err;
                bp.fallbacks = ctx->fallbacks;
                bp.N = N;
                bp.T = plan_of(ctx).big_tiles;
                bp.J = J;
                bp.R = R;
                bp.G = ctx->bigx_grid;
                bp.lam = s->forgetting;
                bp.eps = eps;
                bp.pass = pass;
                bp.final_pass = last;
                bp.post_wait = 0;  // the F GEMM runs between k_bigx and k_bigx_post (it waits for k_bigx)
                if (launch_bigx(ctx, st, b, bp)) return DASH_E_CUDA;
            }
        }
        if (ctx->smallx) {
            // F and G of the small slices: X^T US and US^T US over the small-slice tiles
            if constexpr (!f32)
                if (launch_f3(ctx, st, b, J, (const double *)ctx->us.p, R, Fsl,
                              ctx->bigx ? (const uint32_t *)ctx->tflag.p : nullptr, Gsl))
                    return DASH_E_CUDA;
        } else if (ctx->tma) {
            if (launch_f3(ctx, st, b, J, (const double *)ctx->us.p, R, Fsl,
                          ctx->bigx ? (const uint32_t *)ctx->tflag.p : nullptr))
                return DASH_E_CUDA;
        } else if (ctx->stream) {
            if constexpr (!f32) {
                if (rank_bucket(R) <= 8) launch_f2_t<8>(ctx, st, b, J, (const double *)ctx->us.p, R, Fsl);
                else launch_f2_t<16>(ctx, st, b, J, (const double *)ctx->us.p, R, Fsl);
            }
        } else if (ctx->wtma) {
            if (launch_fw(ctx, st, b, J, (const double *)ctx->us.p, R, Fsl, ctx->swide ? Gsl : nullptr))
                return DASH_E_CUDA;
        } else {
            launch_fgemm(ctx, st, b, J, Ud, (const int32_t *)ctx->row_slice.p, s->W, R, ctx->rps,
                         (int)ctx->nsplit, Fsl, ctx->swide ? Gsl : nullptr);
        }
        // big slices' S-row systems and F / G slots: beside the F GEMM (independent of it)
        if (ctx->bigx && launch_bigx_post(ctx, st, bp)) return DASH_E_CUDA;
    }
    if constexpr (f32) {
        if (last && N > 0) {
            const int64_t n = N * R;
            k_u_to_f32<<<(int)std::min<int64_t>((n + 255) / 256, (int64_t)ctx->num_sms * 8), 256, 0, st>>>(
                Ud, n, (float *)U_out);
            ctx->last_launches++;
        }
    }
    if (host_timing) fprintf(stderr, "[dash host] pass_begin total %.1f us\n", std::chrono::duration<double, std::micro>(tnow() - t0).count());
    {
        PhaseScope ps(ctx, st, PH_SUMFG);
        if (colsum2(ctx, st, Fsl, N > 0 ? (ctx->smallx ? ctx->sx_grid : (int)ctx->nsplit) + ctx->bigx_nbig : 0,
                    (int64_t)J * R, fg_out, Gsl,
                    N > 0 ? ctx->nitems : 0, (int64_t)R * R, fg_out + (int64_t)J * R))
            return DASH_E_CUDA;
    }
    return cudaGetLastError() == cudaSuccess ? DASH_OK : DASH_E_CUDA;
}

extern "C" {

int dash_ctx_create(dash_ctx **out) {
    if (!out) return DASH_E_ARG;
    dash_ctx *ctx = new dash_ctx();
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaMalloc(&ctx->err, sizeof(unsigned long long)) != cudaSuccess ||
        cudaMalloc(&ctx->fallbacks, sizeof(unsigned int)) != cudaSuccess ||
        cudaMalloc(&ctx->vs_flag, sizeof(unsigned int)) != cudaSuccess) {
        delete ctx;
        return DASH_E_CUDA;
    }
    unsigned long long none = ~0ull;
    cudaMemcpy(ctx->err, &none, sizeof(none), cudaMemcpyHostToDevice);
    cudaMemset(ctx->fallbacks, 0, sizeof(unsigned int));
    cudaMemset(ctx->vs_flag, 0, sizeof(unsigned int));
    for (int i = 0; i < 2; ++i) cudaEventCreateWithFlags(&ctx->staged[i], cudaEventDisableTiming);
    *out = ctx;
    return DASH_OK;
}

void dash_ctx_destroy(dash_ctx *ctx) {
    if (!ctx) return;
    cudaDeviceSynchronize();
    dash_ctx::Buf *bufs[] = {&ctx->xv,  &ctx->row_slice, &ctx->items, &ctx->gslots, &ctx->fslots,
                             &ctx->vtv, &ctx->fsnap,     &ctx->gsnap, &ctx->fg,     &ctx->part, &ctx->us, &ctx->scratch,
                             &ctx->smeta, &ctx->plan_hist, &ctx->u64,
                             &ctx->tflag, &ctx->bx_ms, &ctx->bx_toff, &ctx->bx_parts,
                             &ctx->sx_tmp, &ctx->sx_units, &ctx->sx_meta, &ctx->rerr};
    for (auto *b : bufs)
        if (b->p) cudaFree(b->p);
    cudaFree(ctx->err);
    cudaFree(ctx->fallbacks);
    cudaFree(ctx->vs_flag);
    for (int i = 0; i < 2; ++i) {
        if (ctx->items_host[i]) cudaFreeHost(ctx->items_host[i]);
        cudaEventDestroy(ctx->staged[i]);
    }
    for (auto e : ctx->ev_pool) cudaEventDestroy(e);
    for (auto &m : ctx->mring) {
        if (m.copied) cudaEventDestroy(m.copied);
        if (m.done) cudaEventDestroy(m.done);
    }
    if (ctx->meta_stream) cudaStreamDestroy(ctx->meta_stream);
    if (ctx->aux_stream) cudaStreamDestroy(ctx->aux_stream);
    for (auto e : {ctx->aux_fork, ctx->aux_join})
        if (e) cudaEventDestroy(e);
    for (auto e : {ctx->plan_ev, ctx->pset_free, ctx->pset_alt.free_ev})
        if (e) cudaEventDestroy(e);
    for (auto *b : {&ctx->pset_alt.smeta, &ctx->pset_alt.plan_hist, &ctx->pset_alt.tflag})
        if (b->p) cudaFree(b->p);
    delete reinterpret_cast<SlicePlan *>(ctx->plan_p);
    delete ctx;
}

int dash_ctx_status(dash_ctx *ctx, void *stream, int64_t *fail_slice_host) {
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaStreamSynchronize(st) != cudaSuccess) return DASH_E_CUDA;
    unsigned long long key = 0;
    if (cudaMemcpy(&key, ctx->err, sizeof(key), cudaMemcpyDeviceToHost) != cudaSuccess) return DASH_E_CUDA;
    unsigned long long none = ~0ull;
    cudaMemcpy(ctx->err, &none, sizeof(none), cudaMemcpyHostToDevice);
    if (key == none) {
        if (fail_slice_host) *fail_slice_host = 0;
        return DASH_OK;
    }
    if (fail_slice_host) {
        long long pos = (long long)(key >> 4);
        *fail_slice_host = pos >= kPosV ? -1 : pos;
    }
    return (int)(key & 15ull);
}

int dash_ctx_last_launches(const dash_ctx *ctx) { return ctx ? ctx->last_launches : 0; }

// debug builds (-DDASH_SX_TRACE): copy k_smallx's per-unit event clocks to the host
int dash_sx_trace(long long *out, int n) {
#ifdef DASH_SX_TRACE
    cudaDeviceSynchronize();
    if (n == -1) return cudaMemcpyFromSymbol(out, g_sxtrace2, sizeof(long long) * 64 * 8 * 8) == cudaSuccess ? 0 : 2;
    return cudaMemcpyFromSymbol(out, g_sxtrace, sizeof(long long) * (size_t)std::min(n, 148 * 64 * 8)) == cudaSuccess
               ? 0
               : DASH_E_CUDA;
#else
    (void)out;
    (void)n;
    return DASH_E_ARG;
#endif
}

int dash_host_row_ptr(const int64_t *counts, int64_t M, int64_t *row_ptr, int64_t *N_out) {
    if (M < 0 || (M > 0 && (!counts || !row_ptr))) return DASH_E_ARG;
    int64_t acc = 0, tiles = 0;
    int nbig = 0;
    if (row_ptr) row_ptr[0] = 0;
    for (int64_t m = 0; m < M; ++m) {
        const int64_t c = counts[m];
        if (c < 0) return DASH_E_ARG;
        acc += c;
        row_ptr[m + 1] = acc;
        if (c > kSmallRows) {  // the planner's big-slice count, gathered in the same pass
            ++nbig;
            tiles += (c + kTR - 1) / kTR;
        }
    }
    if (N_out) *N_out = acc;
    g_rp_stats.row_ptr = row_ptr;
    g_rp_stats.M = M;
    g_rp_stats.N = acc;
    g_rp_stats.nbig = nbig;
    g_rp_stats.tiles = tiles;
    return DASH_OK;
}

int dash_meta_ring_set(dash_ctx *ctx, int32_t nslots, void *const *pinned, void *const *device, int64_t cap) {
    if (!ctx || nslots < 1 || nslots > dash_ctx::kMetaSlots || !pinned || !device || cap < 0) return DASH_E_ARG;
    if (!ctx->meta_stream && cudaStreamCreateWithFlags(&ctx->meta_stream, cudaStreamNonBlocking) != cudaSuccess)
        return DASH_E_CUDA;
    for (int i = 0; i < nslots; ++i) {
        dash_ctx::MetaSlot &s = ctx->mring[i];
        s.pin = (uint8_t *)pinned[i];
        s.dev = (uint8_t *)device[i];
        if (!s.copied && (cudaEventCreateWithFlags(&s.copied, cudaEventDisableTiming) != cudaSuccess ||
                          cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming) != cudaSuccess))
            return DASH_E_CUDA;
        s.copy_issued = s.upd_issued = false;
    }
    if (!ctx->plan_ev && (cudaEventCreateWithFlags(&ctx->plan_ev, cudaEventDisableTiming) != cudaSuccess ||
                          cudaEventCreateWithFlags(&ctx->pset_free, cudaEventDisableTiming) != cudaSuccess ||
                          cudaEventCreateWithFlags(&ctx->pset_alt.free_ev, cudaEventDisableTiming) != cudaSuccess))
        return DASH_E_CUDA;
    ctx->mring_n = nslots;
    ctx->mring_i = 0;
    ctx->mring_last = -1;
    ctx->mring_cap = (size_t)cap;
    return DASH_OK;
}

int dash_stage_meta(dash_ctx *ctx, void *stream, const int64_t *counts, int32_t M_old, const int32_t *existing_rows,
                    int32_t L, int32_t K_base, void *keep_dev, dash_staged *out) {
    if (!ctx || !out || ctx->mring_n < 1 || M_old < 0 || L < 0 || (M_old > 0 && !existing_rows)) return DASH_E_ARG;
    const int64_t M = (int64_t)M_old + L;
    const size_t o_sr = 8 * (size_t)(M + 1), o_nw = o_sr + ((4 * (size_t)M + 7) / 8) * 8, nbytes = o_nw + (size_t)M;
    if (nbytes > ctx->mring_cap || (M > 0 && !counts)) return DASH_E_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    const int si = ctx->mring_i;
    dash_ctx::MetaSlot &s = ctx->mring[si];
    ctx->mring_i = (si + 1) % ctx->mring_n;
    if (s.copy_issued && cudaEventSynchronize(s.copied) != cudaSuccess) return DASH_E_CUDA;  // pinned block free again
    int64_t *row_ptr = reinterpret_cast<int64_t *>(s.pin);
    int64_t N = 0;
    const int rc = dash_host_row_ptr(counts, M, row_ptr, &N);
    if (rc != DASH_OK) return rc;
    int32_t *sr = reinterpret_cast<int32_t *>(s.pin + o_sr);
    if (M_old) memcpy(sr, existing_rows, sizeof(int32_t) * (size_t)M_old);
    for (int32_t j = 0; j < L; ++j) sr[M_old + j] = K_base + j;
    if (M_old) memset(s.pin + o_nw, 0, (size_t)M_old);
    if (L) memset(s.pin + o_nw + M_old, 1, (size_t)L);
    if (s.upd_issued && cudaStreamWaitEvent(ctx->meta_stream, s.done, 0) != cudaSuccess) return DASH_E_CUDA;
    if (cudaMemcpyAsync(s.dev, s.pin, nbytes, cudaMemcpyHostToDevice, ctx->meta_stream) != cudaSuccess ||
        cudaEventRecord(s.copied, ctx->meta_stream) != cudaSuccess || cudaStreamWaitEvent(st, s.copied, 0) != cudaSuccess)
        return DASH_E_CUDA;
    s.copy_issued = true;
    if (keep_dev && cudaMemcpyAsync(keep_dev, s.dev, nbytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return DASH_E_CUDA;
    ctx->mring_last = si;
    out->N = N;
    out->M = (int32_t)M;
    out->slot = si;
    out->row_ptr = s.dev;
    out->state_row = s.dev + o_sr;
    out->is_new = s.dev + o_nw;
    out->row_ptr_host = s.pin;
    out->nbytes = (int64_t)nbytes;
    return DASH_OK;
}

int dash_stage_release(dash_ctx *ctx, void *stream) {
    if (!ctx || ctx->mring_last < 0) return DASH_E_ARG;
    dash_ctx::MetaSlot &s = ctx->mring[ctx->mring_last];
    if (cudaEventRecord(s.done, (cudaStream_t)stream) != cudaSuccess) return DASH_E_CUDA;
    s.upd_issued = true;
    return DASH_OK;
}

int dash_ctx_path_flags(const dash_ctx *ctx) {
    if (!ctx) return 0;
    return (ctx->stream ? 1 : 0) | (ctx->tma ? 2 : 0) | (ctx->bigx ? 4 : 0) | (ctx->smallx ? 8 : 0);
}

#ifdef DASH_DEBUG_TIMING
int dash_debug_timing(long long *host, int n) {
    cudaDeviceSynchronize();
    return cudaMemcpyFromSymbol(host, g_dbg, sizeof(long long) * n) == cudaSuccess ? 0 : 2;
}
#endif

int dash_ctx_fallbacks(dash_ctx *ctx, void *stream, int32_t reset) {
    if (!ctx) return -1;
    unsigned int v = 0;
    cudaStream_t st = (cudaStream_t)stream;
    cudaMemcpyAsync(&v, ctx->fallbacks, sizeof(v), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    if (reset) cudaMemsetAsync(ctx->fallbacks, 0, sizeof(unsigned int), st);
    return (int)v;
}

int dash_ctx_set_profiling(dash_ctx *ctx, int enable) {
    if (!ctx) return DASH_E_ARG;
    ctx->prof = enable;
    ctx->ev_recs.clear();
    ctx->ev_used = 0;
    return DASH_OK;
}

int dash_ctx_phase_ms(dash_ctx *ctx, double *ms_out, int32_t *count_out, int32_t nphases) {
    if (!ctx || !ms_out) return DASH_E_ARG;
    for (int i = 0; i < nphases; ++i) {
        ms_out[i] = 0.0;
        if (count_out) count_out[i] = 0;
    }
    for (auto &rec : ctx->ev_recs) {
        cudaEventSynchronize(rec.second.second);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, rec.second.first, rec.second.second);
        if (rec.first < nphases) {
            ms_out[rec.first] += ms;
            if (count_out) count_out[rec.first]++;
        }
    }
    ctx->ev_recs.clear();
    ctx->ev_used = 0;
    return DASH_OK;
}

int dash_update_pass_begin_f64(dash_ctx *ctx, void *stream, const dash_batch_f64 *b, dash_state_f64 *s,
                               double *U_out, double *v_used_out, double eps, int32_t pass, double *fg_out) {
    return pass_begin_impl(ctx, stream, b, s, U_out, v_used_out, eps, pass, fg_out);
}

int dash_update_pass_begin_f32(dash_ctx *ctx, void *stream, const dash_batch_f32 *b, dash_state_f64 *s,
                               float *U_out, double *v_used_out, double eps, int32_t pass, double *fg_out) {
    return pass_begin_impl(ctx, stream, b, s, U_out, v_used_out, eps, pass, fg_out);
}

int dash_update_pass_finish_f64(dash_ctx *ctx, void *stream, dash_state_f64 *s, const double *fg, double eps) {
    if (!ctx || !valid_state(s) || !fg) return DASH_E_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    const int J = s->J, R = s->R;
    switch (rank_bucket(R)) {
        case 4: launch_vsolve_t<4>(ctx, st, fg, s->forgetting, J, R, eps, s->F, s->G, s->V); break;
        case 8: launch_vsolve_t<8>(ctx, st, fg, s->forgetting, J, R, eps, s->F, s->G, s->V); break;
        case 16: launch_vsolve_t<16>(ctx, st, fg, s->forgetting, J, R, eps, s->F, s->G, s->V); break;
        case 32: launch_vsolve_t<32>(ctx, st, fg, s->forgetting, J, R, eps, s->F, s->G, s->V); break;
        default: {
            const size_t smem = sizeof(double) * (64 * SC<64>::LDM + SC<64>::NT + 64);
            ensure_smem_attr(k_vsolve_cta<64>, smem);
            PhaseScope ps(ctx, st, PH_VSOLVE);
            const unsigned int *only_if = nullptr;
            unsigned int gen = 0;
            if (launch_vsolvew<8>(ctx, st, fg, s->forgetting, J, R, eps, s->F, s->G, s->V, gen)) only_if = ctx->vs_flag;
            k_vsolve_cta<64><<<(J + 31) / 32, 256, smem, st>>>(fg, (const double *)ctx->fsnap.p,
                                                               (const double *)ctx->gsnap.p, s->forgetting, J, R, eps,
                                                               s->F, s->G, s->V, ctx->err, ctx->fallbacks, only_if, gen);
            break;
        }
    }
    if (ctx->pset_free && ctx->cur_pass == s->passes - 1) {  // the plan set of this update is free again
        cudaEventRecord(ctx->pset_free, st);
        ctx->pset_used = true;
        // ... and so is the staging slot it read (what dash_stage_release does; the same event serves both)
        if (ctx->mring_last >= 0) {
            dash_ctx::MetaSlot &ms = ctx->mring[ctx->mring_last];
            cudaEventRecord(ms.done, st);
            ms.upd_issued = true;
        }
    }
    return cudaGetLastError() == cudaSuccess ? DASH_OK : DASH_E_CUDA;
}

int dash_update_f64(dash_ctx *ctx, void *stream, const dash_batch_f64 *b, dash_state_f64 *s, double *U_out,
                    double *v_used_out, double eps) {
    if (!ctx || !valid_state(s)) return DASH_E_ARG;
    if (ensure(ctx->fg, sizeof(double) * ((size_t)s->J * s->R + s->R * s->R))) return DASH_E_CUDA;
    double *fg = (double *)ctx->fg.p;
    for (int pass = 0; pass < s->passes; ++pass) {
        int rc = dash_update_pass_begin_f64(ctx, stream, b, s, U_out, v_used_out, eps, pass, fg);
        if (rc) return rc;
        rc = dash_update_pass_finish_f64(ctx, stream, s, fg, eps);
        if (rc) return rc;
    }
    return DASH_OK;
}

int dash_update_f32(dash_ctx *ctx, void *stream, const dash_batch_f32 *b, dash_state_f64 *s, float *U_out,
                    double *v_used_out, double eps) {
    if (!ctx || !valid_state(s)) return DASH_E_ARG;
    if (ensure(ctx->fg, sizeof(double) * ((size_t)s->J * s->R + s->R * s->R))) return DASH_E_CUDA;
    double *fg = (double *)ctx->fg.p;
    for (int pass = 0; pass < s->passes; ++pass) {
        int rc = dash_update_pass_begin_f32(ctx, stream, b, s, U_out, v_used_out, eps, pass, fg);
        if (rc) return rc;
        rc = dash_update_pass_finish_f64(ctx, stream, s, fg, eps);
        if (rc) return rc;
    }
    return DASH_OK;
}

int dash_group_update_f64(dash_ctx *ctx, void *stream, int32_t G, int32_t I, int32_t R, const double *xv,
                          const double *vtv, const double *s_used, const double *c_old, const double *d_old,
                          double lam, double eps, double *u, double *us, double *c_new, double *d_new, double *w,
                          double *g_fresh, int32_t *ok_host) {
    if (!ctx || G < 0 || I < 1 || R < 1 || R > DASH_MAX_RANK) return DASH_E_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    ctx->last_launches = 0;
    const int RB = rank_bucket(R);
    // synthetic batch: slice g owns rows g*I..(g+1)*I of xv; state row g
    std::vector<int64_t> rp(G + 1);
    for (int g = 0; g <= G; ++g) rp[g] = (int64_t)g * I;
    std::vector<int4> items;
    plan_items(rp.data(), G, items, slices_per_item(RB));
    const int nitems = (int)items.size();
    size_t need = sizeof(int64_t) * (G + 1) + sizeof(int32_t) * G + G + 64;
    if (ensure(ctx->scratch, need) || ensure(ctx->gslots, sizeof(double) * std::max(nitems, 1) * R * R))
        return DASH_E_CUDA;
    int64_t *d_rp = (int64_t *)ctx->scratch.p;
    int32_t *d_sr = (int32_t *)(d_rp + G + 1);
    uint8_t *d_new_flag = (uint8_t *)(d_sr + G);
    std::vector<int32_t> sr(G);
    for (int g = 0; g < G; ++g) sr[g] = g;
    cudaMemcpyAsync(d_rp, rp.data(), sizeof(int64_t) * (G + 1), cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_sr, sr.data(), sizeof(int32_t) * G, cudaMemcpyHostToDevice, st);
    cudaMemsetAsync(d_new_flag, 0, G, st);
    // state copies: W <- s_used, C <- c_old, D <- d_old (outputs double as state)
    cudaMemcpyAsync(w, s_used, sizeof(double) * G * R, cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(c_new, c_old, sizeof(double) * G * R, cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(d_new, d_old, sizeof(double) * G * R * R, cudaMemcpyDeviceToDevice, st);
    unsigned int zero = 0;
    cudaMemcpyAsync(ctx->fallbacks, &zero, sizeof(zero), cudaMemcpyHostToDevice, st);
    if (nitems > 0 && stage_items(ctx, st, items)) return DASH_E_CUDA;
    if (G > 0) {
        SliceParams sp;
        sp.items = (const int4 *)ctx->items.p;
        sp.row_ptr = d_rp;
        sp.state_row = d_sr;
        sp.is_new = d_new_flag;
        sp.XV = xv;
        sp.U = u;
        sp.US = nullptr;
        sp.W = w;
        sp.C = c_new;
        sp.D = d_new;
        sp.vtv = vtv;
        sp.G_slots = (double *)ctx->gslots.p;
        sp.err = ctx->err;
        sp.fallbacks = ctx->fallbacks;
        sp.R = R;
        sp.lam = lam;
        sp.eps = eps;
        sp.pass = 1;  // read s from W (= s_used), not the new-slice bootstrap
        sp.final_pass = 1;
        if (dispatch_slices(ctx, st, RB, nitems, sp)) return DASH_E_CUDA;
        k_us<<<std::max(1, std::min(1024, (int)(((int64_t)G * I * R + 255) / 256))), 256, 0, st>>>(u, w, G, I, R, us);
        ctx->last_launches++;
    }
    k_sum_slots<<<(R * R + 255) / 256, 256, 0, st>>>((double *)ctx->gslots.p, G > 0 ? nitems : 0, R * R, g_fresh);
    ctx->last_launches++;
    unsigned int fb = 0;
    cudaMemcpyAsync(&fb, ctx->fallbacks, sizeof(fb), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    if (ok_host) *ok_host = fb == 0 ? 1 : 0;
    return cudaGetLastError() == cudaSuccess ? DASH_OK : DASH_E_CUDA;
}

}  // extern "C"

#include "dash_aux.cuh"
#include "dash_als.cuh"
