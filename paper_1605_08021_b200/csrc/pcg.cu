// pcg.cu -- batched, projected Sternheimer solves (Eq. eqncompressU) and W (Eq. eqnW).
//
// Q(eps~_c - H)Q zeta~_{c mu} = Q xi_mu for all (c, mu).  The solver
// works on the equivalent SPD system Q(H - eps~_c)Q x = -Q xi on range(Q) with
// preconditioned CG (PAPER.md:426 leaves the solver open; H - eps~_c is positive
// on range(Q) because every node lies in [eps_1, eps_Nocc] below the gap).
// Preconditioner: z = Q M r, M = IFFT (|k|^2/2 + tau)^{-1} FFT (Fourier diagonal).
//
// One CG iteration over the whole batch = 6 launches (the CG scalars run inside K2):
//   K1 y = (H - eps_c) p  (+ p.y)          K2 C  = dV Psi^T y, alpha = rz / p.y (hook)
//   K3 Ap = y - Psi C ; x += alpha p ; r -= alpha Ap
//   K1 zh = M r (+ r.zh, r.r)               K2 Cz = dV Psi^T zh, convergence / beta (hook)
//   K3 p = (zh - Psi Cz) + beta p
// The iteration loop is one CUDA graph whose while node re-runs a 4-iteration body until every
// column has converged (device-side condition, no host round trips).
// p.y equals p.Q(H-eps)Q p and r.zh equals r.z because p, r stay in range(Q).
// Per-column activity flags freeze converged columns; every reduction has a
// fixed order, so results do not depend on scheduling.
#include "gemm.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

namespace acp {

// Chebyshev nodes on [eps_1, eps_N] and Lagrange weights
// L[i + c*n_occ] = prod_{c' != c} (eps_i - node_c') / (node_c - node_c').
__global__ void k_cheb(const double* __restrict__ eps, int n_occ, int nc, double* __restrict__ nodes,
                       double* __restrict__ L) {
    __shared__ double sn[256];
    const double e1 = eps[0], eN = eps[n_occ - 1];
    for (int c = threadIdx.x; c < nc; c += blockDim.x) {
        const double th = ((double)c + 0.5) / (double)nc;  // theta_c / pi, c = 1..Nc -> (c - 1/2)/Nc
        const double v = 0.5 * (e1 + eN) + 0.5 * (e1 - eN) * cospi(th);
        sn[c] = v;
        nodes[c] = v;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < n_occ * nc; idx += blockDim.x) {
        const int i = idx % n_occ, c = idx / n_occ;
        double l = 1.0;
        for (int cp = 0; cp < nc; ++cp)
            if (cp != c) l *= (eps[i] - sn[cp]) / (sn[c] - sn[cp]);
        L[idx] = l;
    }
}

__global__ void k_batch_shift(const double* __restrict__ nodes, int nc, int nmu_p, double* __restrict__ shift) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < nc * nmu_p) shift[j] = nodes[j / nmu_p];
}

// R[:, c*nmu_p + mu] = rhs[:, mu]; X = 0.
__global__ void k_pcg_init(int Ng, int nc, int nmu_p, const double* __restrict__ rhs, double* __restrict__ R,
                           double* __restrict__ X) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    size_t tot = (size_t)Ng * nc * nmu_p;
    if (i >= tot) return;
    size_t col = i / Ng, r = i % Ng;
    int mu = (int)(col % nmu_p);
    R[i] = rhs[(size_t)mu * Ng + r];
    X[i] = 0.0;
}

enum { SC_INIT = 0, SC_ALPHA = 1, SC_BETA = 2, SC_WARM = 3 };

struct PcgScal {
    double* rz;      // r.z (current)
    double* bb;      // ||b||^2
    double* alpha;
    double* beta;
    double* res;     // final relative residual
    int* active;
    int* iters;
    const double* dots;  // from K1: [2j] x.y, [2j+1] x.x
};

// Per-column CG scalar recurrences, run once per column inside the K2 GEMM (hook).
struct ScalHook {
    int mode;
    PcgScal s;
    double tol2;
    int n_valid_mu;
    int nmu_p;
    // warm start (node sweep): ||b||^2 per mu, from the first node's cold start; SC_INIT then also
    // tests the warm residual against the tolerance.  nullptr: cold start (r0 = b).
    const double* bb0;
    __device__ __forceinline__ bool tile_active(int n0, int n) const { return tile_active_w(n0, n, 32); }
    __device__ __forceinline__ bool tile_active_w(int n0, int n, int w) const {
        if (mode == SC_INIT || mode == SC_WARM) return true;
        int a = 0;
        for (int c = n0; c < min(n, n0 + w); ++c) a |= s.active[c];
        return a != 0;
    }
    __device__ __forceinline__ void operator()(int j) const {
        if (mode == SC_WARM) return;  // alpha = 1, active = 1 were set by k_warm_set
        if (mode == SC_INIT) {
            const double rz = s.dots[2 * j], rr = s.dots[2 * j + 1];
            const double bb = bb0 ? bb0[j % nmu_p] : rr;
            const bool valid = (j % nmu_p) < n_valid_mu && bb > 0.0;
            s.rz[j] = rz;
            s.bb[j] = bb;
            s.active[j] = (valid && (!bb0 || rr > tol2 * bb)) ? 1 : 0;
            s.iters[j] = 0;
            s.res[j] = (bb0 && bb > 0.0) ? sqrt(rr / bb) : 0.0;
            s.alpha[j] = 0.0;
            s.beta[j] = 0.0;
        } else if (mode == SC_ALPHA) {
            if (s.active[j]) s.alpha[j] = s.rz[j] / s.dots[2 * j];
        } else {
            if (s.active[j]) {
                const double rzn = s.dots[2 * j], rr = s.dots[2 * j + 1];
                s.iters[j] += 1;
                s.res[j] = sqrt(rr / s.bb[j]);
                if (rr <= tol2 * s.bb[j]) {
                    s.active[j] = 0;
                } else {
                    s.beta[j] = rzn / s.rz[j];
                    s.rz[j] = rzn;
                }
            }
        }
    }
};

// K3 after H p: Ap = Y - Psi C;  R -= alpha Ap.  (X += alpha P is deferred to EpBeta of the same
// iteration, which reads P anyway: 24 instead of 48 bytes per element here, 40 instead of 24
// there; the iteration at which a column converges skips EpBeta, so k_pcg_x_final applies that
// last alpha P after the loop -- the same operations on the same values, bitwise the same X.)
struct EpAlpha {
    const double* Y;
    double* R;
    const double* alpha;
    const int* active;
    int ld;
    struct Regs {
        double y, r;
        bool on;
    };
    __device__ __forceinline__ void load(int r, int c, Regs& g) const {
        g.on = active[c] != 0;
        if (!g.on) return;
        const size_t o = (size_t)c * ld + r;
        g.y = Y[o];
        g.r = R[o];
    }
    __device__ __forceinline__ void store(int r, int c, double acc, const Regs& g) const {
        if (!g.on) return;
        R[(size_t)c * ld + r] = g.r - alpha[c] * (g.y - acc);
    }
};
// K3 after M r: Z = Zh - Psi Cz;  X += alpha P;  P = Z + beta P.
struct EpBeta {
    const double* Zh;
    double* P;
    double* X;
    const double* alpha;
    const double* beta;
    const int* active;
    int ld;
    struct Regs {
        double zh, p, x;
        bool on;
    };
    __device__ __forceinline__ void load(int r, int c, Regs& g) const {
        g.on = active[c] != 0;
        if (!g.on) return;
        const size_t o = (size_t)c * ld + r;
        g.zh = Zh[o];
        g.p = P[o];
        g.x = X[o];
    }
    __device__ __forceinline__ void store(int r, int c, double acc, const Regs& g) const {
        if (!g.on) return;
        const size_t o = (size_t)c * ld + r;
        X[o] = g.x + alpha[c] * g.p;
        P[o] = (g.zh - acc) + beta[c] * g.p;
    }
};
// The same two updates with X += alpha P in EpAlpha (EpAlphaX / EpBetaP): used where K3 is bound by
// the DMMA work (N_occ >= 64), where the longer EpBeta epilogue cost more than the saved bytes
// (c4g, 4096 columns: EpBeta + EpAlpha 11.72 ms with X in EpBeta, 11.28 ms here); for N_occ < 64
// K3 is HBM-bound and 64 instead of 72 bytes per element and iteration win.
struct EpAlphaX {
    const double* Y;
    const double* P;
    double* X;
    double* R;
    const double* alpha;
    const int* active;
    int ld;
    struct Regs {
        double y, p, x, r;
        bool on;
    };
    __device__ __forceinline__ void load(int r, int c, Regs& g) const {
        g.on = active[c] != 0;
        if (!g.on) return;
        const size_t o = (size_t)c * ld + r;
        g.y = Y[o];
        g.p = P[o];
        g.x = X[o];
        g.r = R[o];
    }
    __device__ __forceinline__ void store(int r, int c, double acc, const Regs& g) const {
        if (!g.on) return;
        const size_t o = (size_t)c * ld + r;
        const double a = alpha[c];
        X[o] = g.x + a * g.p;
        R[o] = g.r - a * (g.y - acc);
    }
};
struct EpBetaP {
    const double* Zh;
    double* P;
    const double* beta;
    const int* active;
    int ld;
    struct Regs {
        double zh, p;
        bool on;
    };
    __device__ __forceinline__ void load(int r, int c, Regs& g) const {
        g.on = active[c] != 0;
        if (!g.on) return;
        const size_t o = (size_t)c * ld + r;
        g.zh = Zh[o];
        g.p = P[o];
    }
    __device__ __forceinline__ void store(int r, int c, double acc, const Regs& g) const {
        if (!g.on) return;
        P[(size_t)c * ld + r] = (g.zh - acc) + beta[c] * g.p;
    }
};
// Timing probe (acp_kernel_bench which = 4): the K3 main loop with an epilogue that moves no data
// (a store that never fires keeps the accumulators live).
struct EpNull {
    double* sink;
    const int* active;
    struct Regs {
        bool on;
    };
    __device__ __forceinline__ void load(int, int c, Regs& g) const { g.on = active[c] != 0; }
    __device__ __forceinline__ void store(int r, int c, double acc, const Regs& g) const {
        if (g.on && acc == 1.2345e300) sink[(size_t)c + r] = acc;
    }
};
// K3 at the start: P = Z = Zh - Psi Cz (X = 0 stays).
struct EpInit {
    const double* Zh;
    double* P;
    const int* active;
    int ld;
    struct Regs {
        double zh;
        bool on;
    };
    __device__ __forceinline__ void load(int r, int c, Regs& g) const {
        g.on = active[c] != 0;
        if (!g.on) return;
        g.zh = Zh[(size_t)c * ld + r];
    }
    __device__ __forceinline__ void store(int r, int c, double acc, const Regs& g) const {
        if (!g.on) return;
        P[(size_t)c * ld + r] = g.zh - acc;
    }
};

static inline bool pcg_x_in_beta(int n_occ) { return n_occ < 64; }

// After the CG loop: the columns that converged skipped EpBeta in their last iteration, so their
// X lacks that iteration's alpha p (P still holds p, alpha its alpha); still-active columns (max_iter
// reached) had every update.
__global__ void k_pcg_x_final(int Ng, int n, const int* __restrict__ active, const int* __restrict__ iters,
                              const double* __restrict__ alpha, const double* __restrict__ P, double* __restrict__ X) {
    const int c = blockIdx.y;
    if (active[c] || iters[c] == 0) return;
    const double a = alpha[c];
    const size_t o = (size_t)c * Ng;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < Ng; r += gridDim.x * blockDim.x)
        X[o + r] += a * P[o + r];
}

// Resident CTAs per SM requested from ptxas: enough that configs[1]'s 1160 tiles fit one wave
// where the epilogue registers allow it (EpAlpha keeps 2 operands per element, EpBeta 3).
template <class Ep> struct K3Occ { static constexpr int v = 4; };
template <> struct K3Occ<EpBeta> { static constexpr int v = 6; };
template <> struct K3Occ<EpAlpha> { static constexpr int v = 8; };
template <> struct K3Occ<EpBetaP> { static constexpr int v = 8; };
template <> struct K3Occ<EpAlphaX> { static constexpr int v = 6; };

template <class Ep, int OCC = K3Occ<Ep>::v>
__global__ void __launch_bounds__(128, OCC) k_pcg_update(int M, int K, int n, const double* __restrict__ A, int lda,
                                                       const double* __restrict__ B, int ldb, Ep ep) {
    pdl_wait();
    pdl_trigger();
    // skip tiles whose columns are all inactive (uniform per CTA)
    const int n0 = blockIdx.y * NP_BN;
    __shared__ int any;
    if (threadIdx.x == 0) {
        int a = 0;
        for (int c = n0; c < min(n, n0 + NP_BN); ++c) a |= ep.active[c];
        any = a;
    }
    __syncthreads();
    if (!any) return;
    nn_tile_pf(M, K, n, A, lda, B, ldb, blockIdx.x * NP_BM, n0, ep);
}

// Large-K variant (N_occ >= 64): 64 x 64 tiles, multistage cp.async, 256 threads.
template <class Ep, int EPI = 0, int ST = GB_ST, int MINB = 2>
__global__ void __launch_bounds__(256, MINB) k_pcg_update_big(int M, int K, int n, const double* __restrict__ A, int lda,
                                                        const double* __restrict__ B, int ldb, Ep ep) {
    pdl_wait();
    pdl_trigger();
    const int n0 = blockIdx.y * GB_BN;
    __shared__ int any;
    if (threadIdx.x == 0) {
        int a = 0;
        for (int c = n0; c < min(n, n0 + GB_BN); ++c) a |= ep.active[c];
        any = a;
    }
    __syncthreads();
    if (!any) return;
    nn_tile_big<Ep, EPI, ST>(M, K, n, A, lda, B, ldb, blockIdx.x * GB_BM, n0, ep);
}

// N_occ >= 128: 128 x 64 tiles (nn_tile_xl), two CTAs per SM.
template <class Ep, int ST = XL_ST, bool SE = false>
__global__ void __launch_bounds__(256, 2) k_pcg_update_xl(int M, int K, int n, const double* __restrict__ A, int lda,
                                                          const double* __restrict__ B, int ldb, Ep ep) {
    pdl_wait();
    pdl_trigger();
    // grouped rasterisation: XL_GM m-tiles (XL_GM x 128 rows of Psi, 4 MB at N_occ = 256) sweep
    // all column tiles together, so Psi is read from HBM once per launch instead of once per column
    // tile (c4g, 4096 columns: 8.6 GB of the kernel's 12.9 GB DRAM reads were Psi re-reads)
    const int mt = (M + XL_BM - 1) / XL_BM, nt = (n + XL_BN - 1) / XL_BN;
    const int b = blockIdx.x, grp = b / (XL_GM * nt), gm0 = grp * XL_GM, gsz = min(XL_GM, mt - gm0);
    const int loc = b - grp * XL_GM * nt;
    const int m0 = (gm0 + loc % gsz) * XL_BM, n0 = (loc / gsz) * XL_BN;
    __shared__ int any;
    if (threadIdx.x == 0) {
        int a = 0;
        for (int c = n0; c < min(n, n0 + XL_BN); ++c) a |= ep.active[c];
        any = a;
    }
    __syncthreads();
    if (!any) return;
    nn_tile_xl<Ep, ST, SE>(M, K, n, A, lda, B, ldb, m0, n0, ep);
}

// N_occ >= 64, warp-specialised persistent form of the 128 x 64 tile (nn_ws_persistent).
template <class Ep>
__global__ void __launch_bounds__(WS_T, 1) k_pcg_update_ws(int M, int K, int n, const double* __restrict__ A, int lda,
                                                           const double* __restrict__ B, int ldb, Ep ep) {
    pdl_wait();
    pdl_trigger();
    nn_ws_persistent<Ep>(M, K, n, A, lda, B, ldb, ep);
}

template <class Ep>
static void launch_pcg_update(acp_context* ctx, int M, int K, int n, const double* A, int lda, const double* B,
                              int ldb, const Ep& ep) {
    cudaLaunchConfig_t cfg = {};
    cfg.stream = ctx->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = ctx->pdl ? 1 : 0;
    // 128 x 64 tiles for N_occ >= 128: c4g EpBeta 5.25 vs 5.71 ms, EpAlpha 6.03 vs 7.63 ms per 4096
    // columns, 11.13 vs 12.85 s per step (same box); 4 stages: 5.73 / 7.00 ms
    // (c3g, N_occ = 64: 651 vs 698 ms per step with the 64 x 64 tile)
    static const int xl_mink = getenv("ACP_K3_XL_MINK") ? atoi(getenv("ACP_K3_XL_MINK")) : 64;
    // warp-specialised persistent form for 64 <= N_occ < 256 (same box, ws / xl: c3g EpBeta 2.49 / 2.62,
    // EpAlpha 2.98 / 3.39 ms per 7680 columns; c2 0.276 / 0.302, 0.294 / 0.355 ms per 4096); at N_occ
    // = 256 one CTA of 8 DMMA warps per SM is slower than two XL CTAs (c4g EpBeta 5.90 vs 5.46 ms)
    static const int ws_env = getenv("ACP_K3_WS") ? atoi(getenv("ACP_K3_WS")) : -1;
    const bool ws = ws_env >= 0 ? ws_env != 0 : K < 256;
    if (K >= xl_mink && ws) {
        auto kern = k_pcg_update_ws<Ep>;
        const size_t smem = nn_ws_smem();
        func_attr((const void*)kern, (int)smem);
        int sms = 148;
        ACP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
        const long long tiles = (long long)cdiv(M, XL_BM) * cdiv(n, XL_BN);
        cfg.gridDim = dim3((unsigned)std::min<long long>(sms, tiles), 1, 1);
        cfg.blockDim = dim3(WS_T, 1, 1);
        cfg.dynamicSmemBytes = smem;
        ACP_CUDA(cudaLaunchKernelEx(&cfg, kern, M, K, n, A, lda, B, ldb, ep));
    } else if (K >= xl_mink) {
        // staged epilogue (accumulators through shared memory, thread = row): c4g 38088 columns EpBeta
        // 48.57 vs 50.39 ms, EpAlpha 50.87 vs 52.96 ms, step 10.12 vs 10.26 s
        static const int se = getenv("ACP_K3_SE") ? atoi(getenv("ACP_K3_SE")) : 1;
        auto kern = se ? k_pcg_update_xl<Ep, 3, true> : k_pcg_update_xl<Ep, 3, false>;
        const size_t smem = nn_xl_smem<3>();
        func_attr((const void*)kern, (int)smem);
        cfg.gridDim = dim3((unsigned)((long long)cdiv(M, XL_BM) * cdiv(n, XL_BN)), 1, 1);
        cfg.blockDim = dim3(256, 1, 1);
        cfg.dynamicSmemBytes = smem;
        ACP_CUDA(cudaLaunchKernelEx(&cfg, kern, M, K, n, A, lda, B, ldb, ep));
    } else if (K >= 64) {
        // epilogue order 1 (nn_tile_big: both halves loaded after the K loop), same-box A/B:
        // configs[3] 836.8 / 824.9 / 828.2 ms and configs[2] 252.0 / 251.0 / 252.8 ms per step for
        // orders 0 / 1 / 2; a 2-stage ring with 3 CTAs/SM was slower (804 vs 763 ms, spills)
        auto kern = k_pcg_update_big<Ep, 1>;
        const size_t smem = nn_big_smem();
        func_attr((const void*)kern, (int)smem);
        cfg.gridDim = dim3(cdiv(M, GB_BM), cdiv(n, GB_BN), 1);
        cfg.blockDim = dim3(256, 1, 1);
        cfg.dynamicSmemBytes = smem;
        ACP_CUDA(cudaLaunchKernelEx(&cfg, kern, M, K, n, A, lda, B, ldb, ep));
    } else {
        cfg.gridDim = dim3(cdiv(M, NP_BM), cdiv(n, NP_BN), 1);
        cfg.blockDim = dim3(128, 1, 1);
        cfg.dynamicSmemBytes = 0;
        ACP_CUDA(cudaLaunchKernelEx(&cfg, k_pcg_update<Ep>, M, K, n, A, lda, B, ldb, ep));
    }
    launched(ctx);
}


// Number of still-active columns; sets the while-node condition of the PCG graph (continue while
// columns remain and fewer than max_chunks chunks ran) and counts the trips.
__global__ void k_count_active(const int* __restrict__ active, int n, int* __restrict__ out,
                               cudaGraphConditionalHandle h, int* __restrict__ chunks, int max_chunks) {
    pdl_wait();
    __shared__ int red[32];
    int s = 0;
    for (int j = threadIdx.x; j < n; j += blockDim.x) s += active[j];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        *out = t;
        const int c = ++(*chunks);
        if (max_chunks > 0) cudaGraphSetConditional(h, (t > 0 && c < max_chunks) ? 1u : 0u);
    }
}

// W(:, mu) = 2f sum_c X(:, c*nmu_p + mu) (.) Phi_c(:, mu),
// Phi_c(alpha, mu) = sum_i Psi(alpha, i) L(i, c) Psi(r_mu, i)   (Eq. eqnW).
// Phi_c = Psi B_c with B_c(i, mu) = L(i, c) Psi(r_mu, i) is a genuine GEMM (N_g x N_occ x N_mu):
// one DMMA GEMM per node whose epilogue accumulates W += 2f X_c (.) Phi_c (nodes in order).
constexpr int W_MAXC = 32;
constexpr int PCG_MAXGRP = 64;  // groups of a sequential node sweep (streams: PCG_MAXG)
constexpr int PCG_SWEEP_DEF = 1;  // nodes per warm-started group of the sweep (A/B: ACP_PCG_SWEEP)
constexpr int PCG_WARM_K = 3;
constexpr double PCG_WARM_TOL = 1.0;  // warm-started groups stop at this fraction of the CG tolerance (A/B)
constexpr int PCG_DEFG = 4;  // default group count for small batches (PCG_MAXG with ACP_PCG_GROUPS)
__global__ void k_w_rhs(int Ng, int n_occ, int nc, int cnt, const double* __restrict__ Psi,
                        const double* __restrict__ L, const int* __restrict__ S, int mu_begin,
                        double* __restrict__ B) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;  // orbital
    const int mu = blockIdx.y, c = blockIdx.z;
    if (i >= n_occ) return;
    B[((size_t)c * cnt + mu) * n_occ + i] = L[c * n_occ + i] * Psi[(size_t)i * Ng + S[mu_begin + mu]];
}

struct EpW {
    const double* X;  // PCG solutions, column c*nmu_p + mu
    double* W;
    int Ng, nmu_p, c, mu_begin;
    double pref;
    int first;
    struct Regs {
        double x, w;
    };
    __device__ __forceinline__ void load(int r, int col, Regs& g) const {
        g.x = X[(size_t)(c * nmu_p + col) * Ng + r];
        g.w = first ? 0.0 : W[(size_t)(mu_begin + col) * Ng + r];
    }
    __device__ __forceinline__ void store(int r, int col, double acc, const Regs& g) const {
        W[(size_t)(mu_begin + col) * Ng + r] = g.w + pref * (g.x * acc);
    }
};

// Node-parallel W (small problems): T_c = 2f X_c (.) (Psi B_c) for all nodes at once (one CTA per
// tile and node), then W = sum_c T_c in node order -- the same additions in the same order as the
// node-sequential epilogue (0 + t_0 + t_1 + ...), so W is bitwise identical.
struct EpWTerm {
    const double* X;
    double* T;  // [c][col][row], ld Ng, cnt columns per node
    int Ng, nmu_p, cnt;
    double pref;
    struct Regs {
        double x;
    };
    __device__ __forceinline__ void load(int r, int col, Regs& g) const {
        g.x = X[(size_t)(blockIdx.z * nmu_p + col) * Ng + r];
    }
    __device__ __forceinline__ void store(int r, int col, double acc, const Regs& g) const {
        T[((size_t)blockIdx.z * cnt + col) * Ng + r] = pref * (g.x * acc);
    }
};
__global__ void k_w_sum(size_t per, int n_cheb, const double* __restrict__ T, double* __restrict__ W) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= per) return;
    double w = 0.0;
    for (int c = 0; c < n_cheb; ++c) w = w + T[(size_t)c * per + i];
    W[i] = w;
}

template <class Ep>
__global__ void __launch_bounds__(128) k_nn_ep(int M, int K, int n, const double* __restrict__ A, int lda,
                                               const double* __restrict__ B, int ldb, Ep ep) {
    nn_tile(M, K, n, A, lda, B, ldb, blockIdx.x * NN_BM, blockIdx.y * NN_BN, ep);
}
template <class Ep>
__global__ void __launch_bounds__(256, 2) k_nn_ep_big(int M, int K, int n, const double* __restrict__ A, int lda,
                                                      const double* __restrict__ B, int ldb, Ep ep) {
    nn_tile_big(M, K, n, A, lda, B, ldb, blockIdx.x * GB_BM, blockIdx.y * GB_BN, ep);
}
__global__ void __launch_bounds__(128) k_w_terms(int M, int K, int n, const double* __restrict__ A,
                                                const double* __restrict__ B, EpWTerm ep) {
    nn_tile_pf(M, K, n, A, M, B + (size_t)blockIdx.z * n * K, K, blockIdx.x * NP_BM, blockIdx.y * NP_BN, ep);
}

// All nodes in ONE launch: each CTA owns a W tile and runs the N_c tile GEMMs in node order,
// accumulating into its W tile (the same thread owns the same element in every pass).
template <bool BIG>
__global__ void __launch_bounds__(BIG ? 256 : 128) k_w_nodes(int M, int K, int n, int n_cheb, const double* __restrict__ A,
                                                             const double* __restrict__ B, EpW ep) {
    for (int c = 0; c < n_cheb; ++c) {
        ep.c = c;
        ep.first = c == 0;
        if (BIG)
            nn_tile_big(M, K, n, A, M, B + (size_t)c * n * K, K, blockIdx.x * GB_BM, blockIdx.y * GB_BN, ep);
        else
            nn_tile(M, K, n, A, M, B + (size_t)c * n * K, K, blockIdx.x * NN_BM, blockIdx.y * NN_BN, ep);
        __syncthreads();
    }
}

template <class Ep>
static void launch_nn_ep(acp_context* ctx, int M, int K, int n, const double* A, int lda, const double* B, int ldb,
                         const Ep& ep) {
    if (K >= 64) {
        func_attr((const void*)k_nn_ep_big<Ep>, (int)nn_big_smem());
        k_nn_ep_big<Ep><<<dim3(cdiv(M, GB_BM), cdiv(n, GB_BN)), 256, nn_big_smem(), ctx->stream>>>(M, K, n, A, lda, B,
                                                                                                   ldb, ep);
    } else {
        k_nn_ep<Ep><<<dim3(cdiv(M, NN_BM), cdiv(n, NN_BN)), 128, 0, ctx->stream>>>(M, K, n, A, lda, B, ldb, ep);
    }
    launched(ctx);
}

// One independent group of columns (a contiguous range of Chebyshev nodes) of the batch: its
// buffers are column slices of the batch's, so groups never touch each other's data.
// Node sweep (warm starts): every column active with alpha = 1 for the residual half-step.
__global__ void k_warm_set(int n, int* __restrict__ active, double* __restrict__ alpha) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n) {
        active[j] = 1;
        alpha[j] = 1.0;
    }
}

// Initial guess for node c from the k solved nodes c0 - k .. c0 - 1: the solution zeta(eps~) of
// Q(H - eps~)Q zeta = Q xi is analytic in eps~ (the premise of Eq. eqnparam's Chebyshev
// interpolation), so the Lagrange polynomial through the solved nodes,
// evaluated at node c, is close to zeta_c.  P_c = sum_i w_i X_i; X_c = the same (xset) or untouched.
constexpr int WARM_KMAX = 8;
__global__ void k_warm_guess(size_t tot, size_t node_stride, int c, int c0, int k, const double* __restrict__ shift_c,
                             const double* __restrict__ X, double* __restrict__ P, double* __restrict__ Xc, int xset) {
    __shared__ double w[WARM_KMAX];
    if (threadIdx.x < k) {
        const int i = c0 - k + threadIdx.x;
        const double x = shift_c[c], xi = shift_c[i];
        double v = 1.0;
        for (int j = c0 - k; j < c0; ++j)
            if (j != i) v *= (x - shift_c[j]) / (xi - shift_c[j]);
        w[threadIdx.x] = v;
    }
    __syncthreads();
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (size_t)gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int q = 0; q < k; ++q) acc += w[q] * X[(size_t)(c0 - k + q) * node_stride + e];
        P[(size_t)c * node_stride + e] = acc;
        if (xset) Xc[(size_t)c * node_stride + e] = acc;
    }
}

struct PcgGroup {
    double *R, *P, *Y, *X, *C, *shift, *dots;
    PcgScal s;
    int n;          // columns
    int* d_nact;    // [0] active columns, [1] while-loop trips
    int* h_nact;    // pinned host copy
    bool synced;    // the host already waited for this group (host-driven loop)
    long long launches_per_trip;
};

// Enqueue the PCG of one group on ctx->stream: r0 = b, z0 = Q M r0, p0 = z0, then the iteration
// loop (while-node graph).  Returns without waiting unless the host-driven loop is selected.
static void pcg_group_enqueue(acp_context* ctx, const double* Psi, int n_occ, const double* V, PcgGroup& G,
                              int nmu_p, double tol2, double tau, int max_iter, const double* bb0 = nullptr) {
    const int Ng = ctx->Ng;
    double *R = G.R, *P = G.P, *Y = G.Y, *X = G.X, *C = G.C, *shift = G.shift, *dots = G.dots;
    PcgScal& s = G.s;
    const int n = G.n;
    int* d_nact = G.d_nact;
    int* h_nact = G.h_nact;
    const int nvalid = nmu_p;  // columns beyond the caller's count are zero RHS -> inactive by bb = 0
    G.synced = false;
    const bool x_in_beta = pcg_x_in_beta(n_occ);

    auto precond_half = [&](int mode) {
        FopArgs f;
        f.X = R;
        f.Y = Y;
        f.n = n;
        f.sym = MULT_PRECOND;  // in-kernel symbol (no table traffic)
        f.tau = tau;
        f.active = (mode == SC_INIT) ? nullptr : s.active;
        f.dots = dots;
        fourier_op(ctx, f);
        const ScalHook hk{mode, s, tol2, nvalid, nmu_p, mode == SC_INIT ? bb0 : nullptr};
        ACP_REQUIRE(launch_tn_cluster(ctx, Ng, n_occ, n, ctx->dV, Psi, Ng, Y, Ng, C, n_occ, hk),
                    "projection GEMM needs an even grid");
        if (mode == SC_INIT) {
            launch_pcg_update(ctx, Ng, n_occ, n, Psi, Ng, C, n_occ, EpInit{Y, P, s.active, Ng});
        } else if (x_in_beta) {
            launch_pcg_update(ctx, Ng, n_occ, n, Psi, Ng, C, n_occ, EpBeta{Y, P, X, s.alpha, s.beta, s.active, Ng});
        } else {
            launch_pcg_update(ctx, Ng, n_occ, n, Psi, Ng, C, n_occ, EpBetaP{Y, P, s.beta, s.active, Ng});
        }
    };
    auto hamiltonian_half = [&](int hmode = SC_ALPHA) {
        FopArgs f;
        f.X = P;
        f.Y = Y;
        f.n = n;
        f.sym = MULT_KINETIC;
        f.diag = V;
        f.shift = shift;
        f.active = s.active;
        f.dots = dots;
        fourier_op(ctx, f);
        const ScalHook hk{hmode, s, tol2, nvalid, nmu_p, nullptr};
        ACP_REQUIRE(launch_tn_cluster(ctx, Ng, n_occ, n, ctx->dV, Psi, Ng, Y, Ng, C, n_occ, hk),
                    "projection GEMM needs an even grid");
        if (x_in_beta)
            launch_pcg_update(ctx, Ng, n_occ, n, Psi, Ng, C, n_occ, EpAlpha{Y, R, s.alpha, s.active, Ng});
        else
            launch_pcg_update(ctx, Ng, n_occ, n, Psi, Ng, C, n_occ, EpAlphaX{Y, P, X, R, s.alpha, s.active, Ng});
    };

    if (bb0) {
        // warm start: P holds the guess x0 (X = x0 too when K3 leaves X to EpBeta, else X = 0), R = b.
        // One Hamiltonian half with alpha = 1 on every column: R = b - Q(H - eps~)Q x0, X = x0.
        k_warm_set<<<cdiv(n, 256), 256, 0, ctx->stream>>>(n, s.active, s.alpha);
        launched(ctx);
        hamiltonian_half(SC_WARM);
    }
    // r0 = b (or the warm residual), z0 = Q M r0, p0 = z0
    precond_half(SC_INIT);

    // The whole iteration loop is ONE CUDA graph with a device-side while node: its body is
    // `chunk` CG iterations + k_count_active, which sets the loop condition (columns still active
    // and fewer than max_iter iterations done) -- no host round trip until every column has
    // converged.  Cached per shapes/pointers; the chunk counter is reset before each launch.
    const int chunk = 4;  // CG iterations per while-node trip (2 / 8: 11.60 / 11.62 vs 11.57 ms/step)
    const int max_chunks = (max_iter + chunk - 1) / chunk;
    int* d_chunks = d_nact + 1;
    char key[512];
    snprintf(key, sizeof(key), "pcgw%d:%d:%d:%d:%d:%d:%d:%.17g:%.17g:%p:%p:%p:%p:%p:%p:%p:%p:%p:%p:%p:%p", chunk, Ng, n,
             n_occ, nmu_p, nvalid, max_chunks, tol2, tau, (void*)Psi, (void*)V, (void*)R, (void*)P, (void*)Y,
             (void*)X, (void*)C, (void*)shift, (void*)dots, (void*)s.rz, (void*)s.active, (void*)d_nact);
    // ACP_PCG_HOSTLOOP=1: the same body as a plain graph replayed from the host (ncu cannot
    // profile kernels inside conditional-node bodies; the launch lists in profiles/ use this)
    if (getenv("ACP_PCG_HOSTLOOP")) key[0] = 'H';
    cudaGraphExec_t exec = nullptr;
    auto it_g = ctx->graphs.find(key);
    bool hostloop = key[0] == 'H';
    if (getenv("ACP_PCG_NOGRAPH")) {  // debug: the same body launched eagerly from the host
        hostloop = true;
        ACP_CUDA(cudaMemsetAsync(d_chunks, 0, sizeof(int), ctx->stream));
        bool conv = false;
        for (int c = 0; c < max_chunks; ++c) {
            for (int it = 0; it < chunk; ++it) {
                hamiltonian_half();
                precond_half(SC_BETA);
            }
            k_count_active<<<1, 256, 0, ctx->stream>>>(s.active, n, d_nact, (cudaGraphConditionalHandle)0, d_chunks,
                                                       -1);
            launched(ctx);
            ACP_CUDA(cudaMemcpyAsync(h_nact, d_nact, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
            ACP_CUDA(cudaStreamSynchronize(ctx->stream));
            if (h_nact[0] == 0) {
                conv = true;
                break;
            }
        }
        h_nact[0] = conv ? 0 : 1;
    } else if (hostloop) {
        ACP_CUDA(cudaMemsetAsync(d_chunks, 0, sizeof(int), ctx->stream));
        exec = graph_cached(ctx, key, [&]() {
            for (int it = 0; it < chunk; ++it) {
                hamiltonian_half();
                precond_half(SC_BETA);
            }
            k_count_active<<<1, 256, 0, ctx->stream>>>(s.active, n, d_nact, (cudaGraphConditionalHandle)0, d_chunks,
                                                       -1);
            launched(ctx);
        });
        bool conv = false;
        for (int c = 0; c < max_chunks; ++c) {
            graph_launch(ctx, key, exec);
            ACP_CUDA(cudaMemcpyAsync(h_nact, d_nact, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
            ACP_CUDA(cudaStreamSynchronize(ctx->stream));
            if (h_nact[0] == 0) {
                conv = true;
                break;
            }
        }
        h_nact[0] = conv ? 0 : 1;
    } else if (it_g != ctx->graphs.end()) {
        exec = it_g->second.exec;
    } else {
        cudaGraph_t g = nullptr;
        ACP_CUDA(cudaGraphCreate(&g, 0));
        cudaGraphConditionalHandle h;
        ACP_CUDA(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t node;
        ACP_CUDA(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        const long long before = ctx->launches;
        ACP_CUDA(cudaStreamBeginCaptureToGraph(ctx->stream, body, nullptr, nullptr, 0,
                                               cudaStreamCaptureModeThreadLocal));
        try {
            // (programmatic dependent launch measured slower on configs[1]: 14.25 vs 13.84-14.03
            // ms/step -- the early-scheduled dependent CTAs take SM slots from the FFT wave)
            ctx->pdl = false;
            for (int it = 0; it < chunk; ++it) {
                hamiltonian_half();
                precond_half(SC_BETA);
            }
            ctx->pdl = false;
            k_count_active<<<1, 256, 0, ctx->stream>>>(s.active, n, d_nact, h, d_chunks, max_chunks);
            launched(ctx);
        } catch (...) {
            ctx->pdl = false;
            cudaGraph_t tmp = nullptr;
            cudaStreamEndCapture(ctx->stream, &tmp);
            cudaGraphDestroy(g);
            throw;
        }
        cudaGraph_t body2 = nullptr;
        ACP_CUDA(cudaStreamEndCapture(ctx->stream, &body2));
        ACP_CUDA(cudaGraphInstantiate(&exec, g, 0));
        cudaGraphDestroy(g);
        auto& ent = ctx->graphs[key];
        ent.exec = exec;
        ent.launches = ctx->launches - before;  // per loop trip; scaled by the trip count below
        ctx->launches = before;
    }
    if (!hostloop) {
        ACP_CUDA(cudaMemsetAsync(d_chunks, 0, sizeof(int), ctx->stream));
        ACP_CUDA(cudaGraphLaunch(exec, ctx->stream));
        ACP_CUDA(cudaMemcpyAsync(h_nact, d_nact, 2 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        G.launches_per_trip = ctx->graphs[key].launches;
    } else {
        G.synced = true;
    }
}

// Device-side PCG statistics for the deferred mode. Layout of the long long array `st`:
//   [0] solves, [1] total iterations, [2] max iterations, [3] launches (graph trips x per-trip),
//   [4] unconverged columns, [5] max relative residual (double bits), [6] LU status,
//   [8 + 2k] iterations of outer iteration k, [9 + 2k] spare.
struct PcgLaunchCounts {
    long long per_trip[PCG_MAXGRP];
};
__global__ void k_pcg_accum_stats(int n, const int* __restrict__ iters, const double* __restrict__ res,
                                  const double* __restrict__ bb, const int* __restrict__ nact, int ngroups,
                                  PcgLaunchCounts lc, int k, long long* __restrict__ st) {
    __shared__ long long r_n[256], r_it[256], r_mx[256];
    __shared__ double r_res[256];
    long long cnt = 0, it = 0, mx = 0;
    double mr = 0.0;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        if (bb[j] <= 0.0) continue;
        cnt += 1;
        it += iters[j];
        mx = max(mx, (long long)iters[j]);
        mr = fmax(mr, res[j]);
    }
    r_n[threadIdx.x] = cnt;
    r_it[threadIdx.x] = it;
    r_mx[threadIdx.x] = mx;
    r_res[threadIdx.x] = mr;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int t = 1; t < blockDim.x; ++t) {
            cnt += r_n[t];
            it += r_it[t];
            mx = max(mx, r_mx[t]);
            mr = fmax(mr, r_res[t]);
        }
        st[0] += cnt;
        st[1] += it;
        st[2] = max(st[2], mx);
        long long launches = 0, unconv = 0;
        for (int g = 0; g < ngroups; ++g) {
            launches += lc.per_trip[g] * nact[2 * g + 1];
            unconv += nact[2 * g];
        }
        st[3] += launches;
        st[4] += unconv;
        const double prev = __longlong_as_double(st[5]);
        st[5] = __double_as_longlong(fmax(prev, mr));
        st[8 + 2 * k] = it;
    }
}

void sternheimer_batch(acp_context* ctx, const double* Psi, int n_occ, const double* V, const double* d_shift_c,
                       int n_c, const double* rhs, int nmu_p, double tol, int max_iter, double tau, double* X,
                       PcgStats* st) {
    const int Ng = ctx->Ng;
    const int n = n_c * nmu_p;
    if (n == 0) return;
    graph_cache_trim(ctx);
    double* R = ctx->wsd("pcg_R", (size_t)Ng * n);
    double* P = ctx->wsd("pcg_P", (size_t)Ng * n);
    double* Y = ctx->wsd("pcg_Y", (size_t)Ng * n);
    double* shift = ctx->wsd("pcg_shift", n);
    double* dots = ctx->wsd("pcg_dots", 2 * (size_t)n);
    double* C = ctx->wsd("pcg_C", (size_t)n_occ * n);
    PcgScal s;
    s.rz = ctx->wsd("pcg_rz", n);
    s.bb = ctx->wsd("pcg_bb", n);
    s.alpha = ctx->wsd("pcg_alpha", n);
    s.beta = ctx->wsd("pcg_beta", n);
    s.res = ctx->wsd("pcg_res", n);
    s.active = ctx->wsi("pcg_active", n);
    s.iters = ctx->wsi("pcg_iters", n);
    s.dots = dots;
    int* d_nact = ctx->wsi("pcg_nact", 2 * PCG_MAXGRP);  // per group: [0] active columns, [1] trips
    int* h_nact = static_cast<int*>(ctx->pinned);
    // Two node groups on two streams: their kernels overlap, filling the latency gaps of each
    // other's small launches (configs[1]: one K1 launch is a single wave of 464 CTAs).
    // ACP_PCG_GROUPS=1 runs the whole batch as one group.
    // Node groups on separate streams: their kernels overlap, filling the latency gaps of each
    // other's small launches (configs[1]: one K1 launch is a single wave of 464 CTAs).  Small
    // batches only (n N_g <= 16M points): configs[1] 12.38 (4 groups) / 12.64 (2) / 13.01 (1)
    // ms/step; configs[2] gains nothing (270.5 / 271.3 / 272.8).  ACP_PCG_GROUPS overrides (each
    // 2D group needs its own FFT intermediate).
    int ngroups = (size_t)n * Ng <= ((size_t)16 << 20) ? std::min(n_c, PCG_DEFG) : 1;
    if (const char* e = getenv("ACP_PCG_GROUPS")) ngroups = std::max(1, std::min(std::min(n_c, PCG_MAXG), atoi(e)));
    if (getenv("ACP_PCG_HOSTLOOP")) ngroups = 1;
    if (ngroups < 1) ngroups = 1;
    // Node sweep (large batches): the nodes are solved `sweep` at a time, one group after the other
    // on the one stream, each later group WARM-STARTED from the Lagrange extrapolation of up to
    // WARM_KMAX already solved nodes (k_warm_guess) -- the same equations to the same tolerance
    // from a closer start: fewer CG iterations per column, every group still thousands of columns
    // wide.  ACP_PCG_SWEEP = nodes per group (0: off, all nodes in one cold-started batch).
    // Measured (runs R6e, R6h; order-3 guess): c4g 8.12 vs 9.87 s per step, c3g 584 vs 617 ms;
    // configs[2] (N_mu' ~ 592: 203.6 cold) 204-219 ms -- no gain below ~768 columns per node.
    int sweep = ((size_t)n * Ng > ((size_t)16 << 20) && n_c >= 3 && nmu_p >= 768) ? PCG_SWEEP_DEF : 0;
    if (const char* e = getenv("ACP_PCG_SWEEP")) sweep = std::max(0, atoi(e));
    if (sweep >= n_c) sweep = 0;
    if (sweep > 0) ngroups = std::min(PCG_MAXGRP, cdiv(n_c, sweep));
    if (sweep > 0) sweep = cdiv(n_c, ngroups);

    k_batch_shift<<<cdiv(n, 256), 256, 0, ctx->stream>>>(d_shift_c, n_c, nmu_p, shift);
    launched(ctx);
    {
        size_t tot = (size_t)Ng * n;
        k_pcg_init<<<cdiv(tot, 256), 256, 0, ctx->stream>>>(Ng, n_c, nmu_p, rhs, R, X);
        launched(ctx);
    }
    const double tol2 = tol * tol;
    PcgGroup grp[PCG_MAXGRP];
    int gc0[PCG_MAXGRP + 1];  // group g: nodes [g n_c / G, (g+1) n_c / G)
    for (int g = 0; g <= ngroups; ++g) gc0[g] = (sweep > 0 ? std::min(n_c, g * sweep) : g * n_c / ngroups) * nmu_p;
    if (sweep > 0)
        fourier_reserve(ctx, sweep * nmu_p, 0);  // the groups run one after the other on intermediate 0
    else
        for (int g = 0; g < ngroups; ++g) fourier_reserve(ctx, gc0[g + 1] - gc0[g], g);  // before any capture
    for (int g = 0; g < ngroups; ++g) {
        const int c0 = gc0[g], cn = gc0[g + 1] - gc0[g];
        PcgGroup& G = grp[g];
        G.R = R + (size_t)c0 * Ng;
        G.P = P + (size_t)c0 * Ng;
        G.Y = Y + (size_t)c0 * Ng;
        G.X = X + (size_t)c0 * Ng;
        G.C = C + (size_t)c0 * n_occ;
        G.shift = shift + c0;
        G.dots = dots + 2 * (size_t)c0;
        G.s = s;
        G.s.rz += c0;
        G.s.bb += c0;
        G.s.alpha += c0;
        G.s.beta += c0;
        G.s.res += c0;
        G.s.active += c0;
        G.s.iters += c0;
        G.s.dots = G.dots;
        G.n = cn;
        G.d_nact = d_nact + 2 * g;
        G.h_nact = h_nact + 2 * g;
        G.launches_per_trip = 0;
    }
    if (sweep > 0) {
        const size_t node_stride = (size_t)Ng * nmu_p;
        // A tighter tolerance for the warm-started groups (ACP_PCG_WARM_TOL < 1) was tried when the
        // order-8 guess missed the W bar on configs[2]; it did not help (the loss came from the
        // extrapolation order, below) and costs 0.7 s per c4g step at 0.1 -- default 1.
        double warm_tol = PCG_WARM_TOL;
        if (const char* e = getenv("ACP_PCG_WARM_TOL")) warm_tol = atof(e);
        // Solved nodes the guess extrapolates from.  High orders predict better but their large
        // alternating weights amplify the solved nodes' own (near-gap) errors into the guess, and
        // the residual test does not see them: configs[2] golden W (4 outers) 3e-10 cold, 3e-10 at
        // k = 2 / 3, 1e-9 at k = 4, 4e-8 at k = 8 (run R6g).  Default 3.  ACP_PCG_WARM_K: A/B.
        int warm_k = PCG_WARM_K;
        if (const char* e = getenv("ACP_PCG_WARM_K")) warm_k = std::max(1, std::min(WARM_KMAX, atoi(e)));
        const int xset = pcg_x_in_beta(n_occ) ? 1 : 0;
        for (int g = 0; g < ngroups; ++g) {
            const int c0 = gc0[g] / nmu_p, c1 = gc0[g + 1] / nmu_p;
            if (g > 0) {
                const int k = std::min(c0, warm_k);
                for (int c = c0; c < c1; ++c) {
                    k_warm_guess<<<148 * 8, 256, 0, ctx->stream>>>(node_stride, node_stride, c, c0, k, d_shift_c, X, P, X,
                                                                    xset);
                    launched(ctx);
                }
            }
            pcg_group_enqueue(ctx, Psi, n_occ, V, grp[g], nmu_p, g > 0 ? tol2 * warm_tol * warm_tol : tol2, tau, max_iter,
                              g > 0 ? s.bb : nullptr);
        }
        if (!grp[ngroups - 1].synced && !ctx->defer) ACP_CUDA(cudaStreamSynchronize(ctx->stream));
    } else if (ngroups == 1) {
        pcg_group_enqueue(ctx, Psi, n_occ, V, grp[0], nmu_p, tol2, tau, max_iter);
        if (!grp[0].synced && !ctx->defer) ACP_CUDA(cudaStreamSynchronize(ctx->stream));
    } else {
        cudaStream_t s0 = ctx->stream;
        ACP_CUDA(cudaEventRecord(ctx->ev_fork, s0));
        for (int g = 1; g < ngroups; ++g) ACP_CUDA(cudaStreamWaitEvent(ctx->gstream[g], ctx->ev_fork, 0));
        try {
            for (int g = 0; g < ngroups; ++g) {
                ctx->stream = g == 0 ? s0 : ctx->gstream[g];
                ctx->f2_alt = g;  // group g's 2D FFT intermediate
                pcg_group_enqueue(ctx, Psi, n_occ, V, grp[g], nmu_p, tol2, tau, max_iter);
            }
        } catch (...) {
            ctx->stream = s0;
            ctx->f2_alt = 0;
            throw;
        }
        ctx->stream = s0;
        ctx->f2_alt = 0;
        for (int g = 1; g < ngroups; ++g) {
            ACP_CUDA(cudaEventRecord(ctx->ev_join[g], ctx->gstream[g]));
            ACP_CUDA(cudaStreamWaitEvent(s0, ctx->ev_join[g], 0));
        }
        if (!ctx->defer) ACP_CUDA(cudaStreamSynchronize(s0));
    }
    if (pcg_x_in_beta(n_occ)) {
        k_pcg_x_final<<<dim3(cdiv(Ng, 1024), n), 256, 0, ctx->stream>>>(Ng, n, s.active, s.iters, s.alpha, P, X);
        launched(ctx);
    }
    // ACP_PCG_ITERS_HIST: per Chebyshev node min / mean / max CG iterations and the share of the
    // tile work (64-column tiles stay live until their slowest column converges) spent on columns
    // that are still active (stderr; diagnostics only, forces a host wait)
    static const bool iters_hist = getenv("ACP_PCG_ITERS_HIST") != nullptr;
    if (iters_hist) {
        ACP_CUDA(cudaStreamSynchronize(ctx->stream));
        std::vector<int> it(n);
        ACP_CUDA(cudaMemcpy(it.data(), s.iters, n * sizeof(int), cudaMemcpyDeviceToHost));
        long long work = 0, tile_work = 0, all_work = 0;
        int gmax = 0;
        for (int c = 0; c < n_c; ++c) {
            int lo = 1 << 30, hi = 0;
            long long sum = 0;
            for (int j = 0; j < nmu_p; ++j) {
                const int v = it[(size_t)c * nmu_p + j];
                lo = std::min(lo, v);
                hi = std::max(hi, v);
                sum += v;
            }
            gmax = std::max(gmax, hi);
            fprintf(stderr, "[acp pcg iters] node %d: min %d mean %.2f max %d\n", c, lo, (double)sum / nmu_p, hi);
        }
        for (int t0 = 0; t0 < n; t0 += 64) {
            int hi = 0;
            for (int j = t0; j < std::min(n, t0 + 64); ++j) {
                hi = std::max(hi, it[j]);
                work += it[j];
            }
            tile_work += (long long)hi * std::min(64, n - t0);
        }
        all_work = (long long)gmax * n;
        fprintf(stderr, "[acp pcg iters] n %d: column-iterations %lld, 64-column tile work %lld (%.3f useful), no-skip work %lld\n",
                n, work, tile_work, (double)work / (double)tile_work, all_work);
    }
    if (ctx->defer) {
        // no host wait: accumulate the statistics on the device (read at the end of acp_dyson)
        long long lpt[PCG_MAXGRP] = {};
        for (int g = 0; g < ngroups; ++g) lpt[g] = grp[g].synced ? 0 : grp[g].launches_per_trip;
        PcgLaunchCounts lc;
        for (int g = 0; g < PCG_MAXGRP; ++g) lc.per_trip[g] = lpt[g];
        k_pcg_accum_stats<<<1, 256, 0, ctx->stream>>>(n, s.iters, s.res, s.bb, d_nact, ngroups, lc,
                                                        ctx->defer_iter, ctx->defer_stats);
        launched(ctx);
        return;
    }
    bool converged = true;
    for (int g = 0; g < ngroups; ++g) {
        if (!grp[g].synced) ctx->launches += grp[g].launches_per_trip * grp[g].h_nact[1];
        converged = converged && grp[g].h_nact[0] == 0;
    }
    if (st) {
        std::vector<int> it(n);
        std::vector<double> res(n), bb(n);
        ACP_CUDA(cudaMemcpy(it.data(), s.iters, n * sizeof(int), cudaMemcpyDeviceToHost));
        ACP_CUDA(cudaMemcpy(res.data(), s.res, n * sizeof(double), cudaMemcpyDeviceToHost));
        ACP_CUDA(cudaMemcpy(bb.data(), s.bb, n * sizeof(double), cudaMemcpyDeviceToHost));
        for (int j = 0; j < n; ++j) {
            if (bb[j] <= 0.0) continue;
            st->n_solved += 1;
            st->total_iter += it[j];
            if (it[j] > st->max_iter) st->max_iter = it[j];
            if (res[j] > st->max_rel_res) st->max_rel_res = res[j];
        }
    }
    if (!converged)
        throw Error(ACP_ERR_NOT_CONVERGED, "Sternheimer PCG did not converge in " + std::to_string(max_iter) +
                                               " iterations");
}

void apply_chi0(acp_context* ctx, const double* Psi, const double* eps, const double* V, const int* S,
                const double* Xi, int n_mu, int mu_begin, int mu_end, int n_cheb, double tol, int max_iter,
                double* W, PcgStats* st) {
    const int Ng = ctx->Ng;
    const int n_occ = ctx->sys.n_occ;
    ACP_REQUIRE(0 <= mu_begin && mu_begin <= mu_end && mu_end <= n_mu, "invalid mu range");
    ACP_REQUIRE(n_cheb >= 1 && n_cheb <= W_MAXC, "n_cheb must be in [1, 32]");
    ACP_REQUIRE(n_occ <= 256 && n_cheb <= 256, "n_occ too large");
    const int cnt = mu_end - mu_begin;
    if (cnt == 0) return;
    const int nmu_p = (cnt + 1) / 2 * 2;
    double* nodes = ctx->wsd("chi_nodes", n_cheb);
    double* L = ctx->wsd("chi_L", (size_t)n_occ * n_cheb);
    k_cheb<<<1, 256, 0, ctx->stream>>>(eps, n_occ, n_cheb, nodes, L);
    launched(ctx);
    // rhs_mu = -Q xi_mu  (Q xi = xi - Psi dV Psi^T xi), padded with a zero column.
    double* rhs = ctx->wsd("chi_rhs", (size_t)Ng * nmu_p);
    double* Cb = ctx->wsd("chi_Cb", (size_t)n_occ * nmu_p);
    if (nmu_p != cnt) fill(ctx, rhs + (size_t)cnt * Ng, Ng, 0.0);
    copy_cols(ctx, rhs, Xi + (size_t)mu_begin * Ng, (size_t)cnt * Ng);
    gemm_tn(ctx, Ng, n_occ, cnt, ctx->dV, Psi, Ng, rhs, Ng, Cb);
    gemm_nn(ctx, Ng, n_occ, cnt, 1.0, Psi, Ng, Cb, n_occ, -1.0, rhs, Ng);
    double* X = ctx->wsd("chi_X", (size_t)Ng * n_cheb * nmu_p);
    const double tau = 0.05;
    sternheimer_batch(ctx, Psi, n_occ, V, nodes, n_cheb, rhs, nmu_p, tol, max_iter, tau, X, st);
    double* B = ctx->wsd("chi_Bw", (size_t)n_cheb * cnt * n_occ);
    k_w_rhs<<<dim3(cdiv(n_occ, 128), cnt, n_cheb), 128, 0, ctx->stream>>>(Ng, n_occ, n_cheb, cnt, Psi, L, S, mu_begin,
                                                                         B);
    launched(ctx);
    EpW ep{X, W, Ng, nmu_p, 0, mu_begin, 2.0 * ctx->sys.occ, 1};
    if (n_occ < 64 && (size_t)n_cheb * cnt * Ng * sizeof(double) <= ((size_t)256 << 20) &&
               !getenv("ACP_W_SEQ")) {
        // small problems (configs[1]): all nodes in parallel, then the ordered sum
        double* T = ctx->wsd("chi_Wterms", (size_t)n_cheb * cnt * Ng);
        EpWTerm et{X, T, Ng, nmu_p, cnt, 2.0 * ctx->sys.occ};
        k_w_terms<<<dim3(cdiv(Ng, NP_BM), cdiv(cnt, NP_BN), n_cheb), 128, 0, ctx->stream>>>(Ng, n_occ, cnt, Psi, B,
                                                                                           et);
        launched(ctx);
        const size_t per = (size_t)cnt * Ng;
        k_w_sum<<<cdiv((long long)per, 256), 256, 0, ctx->stream>>>(per, n_cheb, T, W + (size_t)mu_begin * Ng);
        launched(ctx);
    } else if (n_occ >= 64) {
        func_attr((const void*)k_w_nodes<true>, (int)nn_big_smem());
        k_w_nodes<true><<<dim3(cdiv(Ng, GB_BM), cdiv(cnt, GB_BN)), 256, nn_big_smem(), ctx->stream>>>(
            Ng, n_occ, cnt, n_cheb, Psi, B, ep);
        launched(ctx);
    } else {
        k_w_nodes<false><<<dim3(cdiv(Ng, NN_BM), cdiv(cnt, NN_BN)), 128, 0, ctx->stream>>>(Ng, n_occ, cnt, n_cheb,
                                                                                          Psi, B, ep);
        launched(ctx);
    }
}

void kernel_bench(acp_context* ctx, int which, const double* Psi, const double* V, const double* X, int n,
                  double* Y, int reps) {
    const int Ng = ctx->Ng, n_occ = ctx->sys.n_occ;
    double* C = ctx->wsd("kb_C", (size_t)n_occ * n);
    double* beta = ctx->wsd("kb_beta", n);
    int* active = ctx->wsi("kb_active", n);
    double* kb_X = which >= 2 ? ctx->wsd("kb_X", (size_t)Ng * n) : nullptr;
    // operand setup once per batch width (outside the caller's timed region on later calls)
    const std::string skey = "kbsetup:" + std::to_string(n);
    if (ctx->graphs.find(skey) == ctx->graphs.end()) {
        fill(ctx, C, (size_t)n_occ * n, 1e-3);
        fill(ctx, beta, n, 0.5);
        std::vector<int> ones(n, 1);  // all columns active
        ACP_CUDA(cudaMemcpyAsync(active, ones.data(), n * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
        ACP_CUDA(cudaStreamSynchronize(ctx->stream));
        ctx->graphs[skey] = acp_context::GraphEntry{};
    }
    fourier_reserve(ctx, n, 0);
    // The reps launches are captured into a CUDA graph (cached per shape) and replayed, so the
    // caller's events time device execution back to back, not host launch overhead.
    auto body = [&]() {
        for (int r = 0; r < reps; ++r) {
            if (which == 0) {
                FopArgs f;
                f.X = X;
                f.Y = Y;
                f.n = n;
                f.sym = MULT_KINETIC;
                f.diag = V;
                f.active = active;
                f.dots = nullptr;
                fourier_op(ctx, f);
            } else if (which == 1) {
                launch_tn_cluster(ctx, Ng, n_occ, n, ctx->dV, Psi, Ng, X, Ng, C, n_occ, NoHook{});
            } else if (which == 2) {
                // the production EpBeta: P = (X - Psi C) + beta P (+ X += alpha P when X is updated there)
                if (pcg_x_in_beta(n_occ))
                    launch_pcg_update(ctx, Ng, n_occ, n, Psi, Ng, C, n_occ, EpBeta{X, Y, kb_X, beta, beta, active, Ng});
                else
                    launch_pcg_update(ctx, Ng, n_occ, n, Psi, Ng, C, n_occ, EpBetaP{X, Y, beta, active, Ng});
            } else if (which == 4) {
                launch_pcg_update(ctx, Ng, n_occ, n, Psi, Ng, C, n_occ, EpNull{Y, active});
            } else {
                // the production EpAlpha: Ap = X - Psi C, R -= alpha Ap (+ X += alpha P)
                if (pcg_x_in_beta(n_occ))
                    launch_pcg_update(ctx, Ng, n_occ, n, Psi, Ng, C, n_occ, EpAlpha{X, Y, beta, active, Ng});
                else
                    launch_pcg_update(ctx, Ng, n_occ, n, Psi, Ng, C, n_occ, EpAlphaX{X, kb_X, kb_X, Y, beta, active, Ng});
            }
        }
    };
    if (getenv("ACP_K1_PROFILE") && which == 0) {
        FopArgs f;
        f.X = X;
        f.Y = Y;
        f.n = n;
        f.sym = MULT_KINETIC;
        f.diag = V;
        f.active = active;
        f.tprof = reinterpret_cast<long long*>(ctx->ws("k1_tprof", 128));
        long long h[16] = {0};
        ACP_CUDA(cudaMemsetAsync(f.tprof, 0, sizeof(h), ctx->stream));
        fourier_op(ctx, f);
        ACP_CUDA(cudaMemcpyAsync(h, f.tprof, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
        ACP_CUDA(cudaStreamSynchronize(ctx->stream));
        fprintf(stderr, "[k1 phase cycles]");
        for (int q = 1; q < 16 && h[q]; ++q) fprintf(stderr, " %lld", h[q] - h[q - 1]);
        fprintf(stderr, "\n");
    }
    char key[256];
    snprintf(key, sizeof(key), "kbench:%d:%d:%d:%p:%p:%p:%p", which, n, reps, (const void*)Psi, (const void*)V,
             (const void*)X, (void*)Y);
    cudaGraphExec_t exec = graph_cached(ctx, key, body);
    graph_launch(ctx, key, exec);
}

}  // namespace acp
