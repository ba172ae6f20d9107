// qrcp.cu -- Alg. 2 with Remark 1 on the GPU.
//
//  K4  G~ = G' Omega            real SRFT of the perturbation columns (DMMA GEMM)
//  K5  M~^T(i + q N_occ, a) = psi_i(a) G~(a, q)   Kronecker rows
//  K6  pivoted QR of M~^T: greedy max-norm pivot among the remaining columns
//      (first index on ties), Householder reflection, trailing update with exact
//      norm recomputation; device-resident (the step index lives in device memory,
//      chunks of steps are replayed from one CUDA graph, no host round trip per pivot)
//  K7  Xi^T = R11^{-1} R_{1:N,:} Pi^{-1} by back substitution + scatter.
#include "gemm.cuh"

#include <cmath>

namespace acp {

// Omega(I, 2q) + i Omega(I, 2q+1) = exp(-2 pi i I nu_q / n) exp(2 pi i theta_I),  I = 1..n.
__global__ void k_srft_omega(int n, int r_half, const double* __restrict__ theta, const int* __restrict__ nu,
                             double* __restrict__ Om) {
    int I0 = blockIdx.x * blockDim.x + threadIdx.x;  // 0-based row
    int q = blockIdx.y;
    if (I0 >= n || q >= r_half) return;
    long long Inu = (long long)(I0 + 1) * (long long)nu[q];
    Inu %= n;
    double frac = theta[I0] - (double)Inu / (double)n;  // turns
    double s, c;
    sincospi(2.0 * frac, &s, &c);
    Om[(size_t)(2 * q) * n + I0] = c;
    Om[(size_t)(2 * q + 1) * n + I0] = s;
}

// A (m x Ng, ld m), m = n_occ * r:  A[i + q n_occ, a] = Psi(a, i) Gt(a, q).  32 grid points per CTA.
__global__ void __launch_bounds__(256) k_kron_rows(int Ng, int n_occ, int r, const double* __restrict__ Psi,
                                                   const double* __restrict__ Gt, double* __restrict__ A) {
    extern __shared__ double sm[];
    double* sp = sm;                 // 32 x n_occ  (a-major)
    double* sg = sm + 32 * n_occ;    // 32 x r
    const int a0 = blockIdx.x * 32;
    for (int idx = threadIdx.x; idx < 32 * n_occ; idx += blockDim.x) {
        int aa = idx % 32, i = idx / 32;
        sp[aa * n_occ + i] = (a0 + aa < Ng) ? Psi[(size_t)i * Ng + a0 + aa] : 0.0;
    }
    for (int idx = threadIdx.x; idx < 32 * r; idx += blockDim.x) {
        int aa = idx % 32, q = idx / 32;
        sg[aa * r + q] = (a0 + aa < Ng) ? Gt[(size_t)q * Ng + a0 + aa] : 0.0;
    }
    __syncthreads();
    const int m = n_occ * r;
    for (int aa = 0; aa < 32 && a0 + aa < Ng; ++aa) {
        double* col = A + (size_t)(a0 + aa) * m;
        for (int idx = threadIdx.x; idx < m; idx += blockDim.x) {
            int i = idx % n_occ, q = idx / n_occ;
            col[idx] = sp[aa * n_occ + i] * sg[aa * r + q];
        }
    }
}

struct QrState {
    int step;      // next pivot step j
    int stop;      // 1 when finished
    int n_mu;      // selected count (valid when stop)
    int kmax;
    double r11;    // |R_11|
};

// norms2[c] = sum_{i >= 0} A[i, c]^2  (warp per column)
__global__ void k_qr_norms(int m, int Ng, const double* __restrict__ A, double* __restrict__ norms2) {
    int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, l = threadIdx.x & 31;
    if (w >= Ng) return;
    const double* col = A + (size_t)w * m;
    double s = 0.0;
    for (int i = l; i < m; i += 32) s += col[i] * col[i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (l == 0) norms2[w] = s;
}

// Single CTA: pivot selection, threshold test, column swap, Householder vector.
__global__ void __launch_bounds__(1024) k_qr_pivot(int m, int Ng, double* __restrict__ A, double* __restrict__ norms2,
                                                   int* __restrict__ perm, double* __restrict__ v, double* __restrict__ tau,
                                                   double* __restrict__ rdiag, QrState* st, double eps, int fixed) {
    __shared__ double sval[32];
    __shared__ int sidx[32];
    __shared__ int s_p;
    __shared__ double s_red[32];
    if (st->stop) return;
    const int j = st->step;
    if (j >= st->kmax) {
        if (threadIdx.x == 0) {
            st->stop = 1;
            st->n_mu = st->kmax;
        }
        return;
    }
    // argmax over c in [j, Ng), first index on ties
    double best = -1.0;
    int bi = Ng;
    for (int c = j + threadIdx.x; c < Ng; c += blockDim.x) {
        double x = norms2[c];
        if (x > best) {  // strictly greater keeps the lowest index within this thread (c increasing)
            best = x;
            bi = c;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        double ob = __shfl_xor_sync(0xffffffffu, best, o);
        int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) {
            best = ob;
            bi = oi;
        }
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        sval[w] = best;
        sidx[w] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double b = -1.0;
        int idx = Ng;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i)
            if (sval[i] > b || (sval[i] == b && sidx[i] < idx)) {
                b = sval[i];
                idx = sidx[i];
            }
        const double rjj = sqrt(b);
        if (j == 0) st->r11 = rjj;
        int stop = 0;
        if (fixed <= 0 && rjj < eps * st->r11) stop = 1;
        if (rjj == 0.0) stop = 1;
        if (stop) {
            st->stop = 1;
            st->n_mu = j;
            s_p = -1;
        } else {
            s_p = idx;
        }
    }
    __syncthreads();
    const int p = s_p;
    if (p < 0) return;
    if (p != j) {
        double* cj = A + (size_t)j * m;
        double* cp = A + (size_t)p * m;
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            double t = cj[i];
            cj[i] = cp[i];
            cp[i] = t;
        }
        if (threadIdx.x == 0) {
            int t = perm[j];
            perm[j] = perm[p];
            perm[p] = t;
            double u = norms2[j];
            norms2[j] = norms2[p];
            norms2[p] = u;
        }
    }
    __syncthreads();
    // Householder: x = A[j:m, j]
    double* cj = A + (size_t)j * m;
    double s = 0.0;
    for (int i = j + threadIdx.x; i < m; i += blockDim.x) s += cj[i] * cj[i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (l == 0) s_red[w] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += s_red[i];
        s_red[0] = t;
    }
    __syncthreads();
    const double xn2 = s_red[0];
    const double xn = sqrt(xn2);
    const double x0 = cj[j];
    const double alpha = (x0 >= 0.0) ? -xn : xn;
    const double v0 = x0 - alpha;
    const double vn2 = xn2 - x0 * x0 + v0 * v0;
    for (int i = j + threadIdx.x; i < m; i += blockDim.x) v[i] = (i == j) ? v0 : cj[i];
    __syncthreads();
    for (int i = j + 1 + threadIdx.x; i < m; i += blockDim.x) cj[i] = 0.0;
    if (threadIdx.x == 0) {
        cj[j] = alpha;
        *tau = (vn2 > 0.0) ? 2.0 / vn2 : 0.0;
        rdiag[j] = xn;
    }
}

// Trailing update for columns c > j (warp per column): A[j:,c] -= tau v (v^T A[j:,c]); new norms (rows > j).
__global__ void __launch_bounds__(256) k_qr_update(int m, int Ng, double* __restrict__ A, double* __restrict__ norms2,
                                                   const double* __restrict__ v, const double* __restrict__ tau,
                                                   QrState* st) {
    if (st->stop) return;
    const int j = st->step;
    const int wpb = blockDim.x >> 5;
    const int l = threadIdx.x & 31;
    const double t = *tau;
    for (int c = j + 1 + blockIdx.x * wpb + (threadIdx.x >> 5); c < Ng; c += gridDim.x * wpb) {
        double* col = A + (size_t)c * m;
        double s = 0.0;
        for (int i = j + l; i < m; i += 32) s += v[i] * col[i];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        const double f = t * s;
        double nn = 0.0;
        for (int i = j + l; i < m; i += 32) {
            double x = col[i] - f * v[i];
            col[i] = x;
            if (i > j) nn += x * x;
        }
        for (int o = 16; o > 0; o >>= 1) nn += __shfl_xor_sync(0xffffffffu, nn, o);
        if (l == 0) norms2[c] = nn;
    }
}

__global__ void k_qr_advance(QrState* st) {
    if (!st->stop) st->step += 1;
}

__global__ void k_iota(int* p, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = i;
}

// T = R11^{-1} R12 (back substitution), one thread per trailing column; T stored row-major (mu, c').
__global__ void k_trsm_cols(int m, int Ng, int N, const double* __restrict__ A, double* __restrict__ T) {
    const int c = N + blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= Ng) return;
    const int nc = Ng - N;
    const int cc = c - N;
    for (int mu = N - 1; mu >= 0; --mu) {
        double s = A[(size_t)c * m + mu];
        for (int nu = mu + 1; nu < N; ++nu) s -= A[(size_t)nu * m + mu] * T[(size_t)nu * nc + cc];
        T[(size_t)mu * nc + cc] = s / A[(size_t)mu * m + mu];
    }
}

// Xi[perm[c], mu] = T[mu, c - N] (c >= N) or delta_{c mu} (c < N);  S[mu] = perm[mu].
__global__ void k_scatter_xi(int Ng, int N, const int* __restrict__ perm, const double* __restrict__ T,
                             double* __restrict__ Xi, int* __restrict__ S) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int mu = blockIdx.y;
    if (c >= Ng) return;
    const int row = perm[c];
    double v;
    if (c < N) v = (c == mu) ? 1.0 : 0.0;
    else v = T[(size_t)mu * (Ng - N) + (c - N)];
    Xi[(size_t)mu * Ng + row] = v;
    if (c == 0) S[mu] = perm[mu];
}

int compress(acp_context* ctx, const double* Psi, const double* Gp, int n_cols, const double* h_theta,
             const int* h_nu, int r_half, double id_eps, int n_fixed, int n_mu_max, int* S, double* Xi) {
    const int Ng = ctx->Ng;
    const int n_occ = ctx->sys.n_occ;
    ACP_REQUIRE(n_cols >= 1 && r_half >= 1 && r_half <= n_cols, "invalid sketch size");
    const int r = 2 * r_half;
    const int m = n_occ * r;
    // Omega from the raw draws
    double* d_theta = ctx->wsd("qr_theta", n_cols);
    int* d_nu = ctx->wsi("qr_nu", r_half);
    ACP_CUDA(cudaMemcpyAsync(d_theta, h_theta, n_cols * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    ACP_CUDA(cudaMemcpyAsync(d_nu, h_nu, r_half * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    double* Om = ctx->wsd("qr_omega", (size_t)n_cols * r);
    k_srft_omega<<<dim3(cdiv(n_cols, 128), r_half), 128, 0, ctx->stream>>>(n_cols, r_half, d_theta, d_nu, Om);
    launched(ctx);
    double* Gt = ctx->wsd("qr_gt", (size_t)Ng * r);
    gemm_nn(ctx, Ng, n_cols, r, 1.0, Gp, Ng, Om, n_cols, 0.0, Gt, Ng);
    // Kronecker rows
    double* A = ctx->wsd("qr_A", (size_t)m * Ng);
    {
        size_t smem = 32 * (size_t)(n_occ + r) * sizeof(double);
        ACP_CUDA(cudaFuncSetAttribute(k_kron_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_kron_rows<<<cdiv(Ng, 32), 256, smem, ctx->stream>>>(Ng, n_occ, r, Psi, Gt, A);
        launched(ctx);
    }
    // QRCP
    int kmax = m < Ng ? m : Ng;
    if (n_fixed > 0 && n_fixed < kmax) kmax = n_fixed;
    if (n_mu_max < kmax && n_fixed > 0) ACP_REQUIRE(false, "n_mu_fixed exceeds n_mu_max");
    double* norms2 = ctx->wsd("qr_norms", Ng);
    int* perm = ctx->wsi("qr_perm", Ng);
    double* v = ctx->wsd("qr_v", m);
    double* tau = ctx->wsd("qr_tau", 1);
    double* rdiag = ctx->wsd("qr_rdiag", kmax);
    QrState* st = static_cast<QrState*>(ctx->ws("qr_state", sizeof(QrState)));
    QrState h0{0, 0, 0, kmax, 0.0};
    ACP_CUDA(cudaMemcpyAsync(st, &h0, sizeof(QrState), cudaMemcpyHostToDevice, ctx->stream));
    k_iota<<<cdiv(Ng, 256), 256, 0, ctx->stream>>>(perm, Ng);
    launched(ctx);
    k_qr_norms<<<cdiv((size_t)Ng * 32, 256), 256, 0, ctx->stream>>>(m, Ng, A, norms2);
    launched(ctx);
    const int upd_blocks = 148 * 4;
    const int chunk = 16;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    long long before = ctx->launches;
    ACP_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    for (int s = 0; s < chunk; ++s) {
        k_qr_pivot<<<1, 1024, 0, ctx->stream>>>(m, Ng, A, norms2, perm, v, tau, rdiag, st, id_eps, n_fixed);
        launched(ctx);
        k_qr_update<<<upd_blocks, 256, 0, ctx->stream>>>(m, Ng, A, norms2, v, tau, st);
        launched(ctx);
        k_qr_advance<<<1, 1, 0, ctx->stream>>>(st);
        launched(ctx);
    }
    ACP_CUDA(cudaStreamEndCapture(ctx->stream, &graph));
    const long long per = ctx->launches - before;
    ctx->launches = before;
    ACP_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    QrState hs{};
    for (int done = 0; done <= kmax + chunk; done += chunk) {
        ACP_CUDA(cudaGraphLaunch(exec, ctx->stream));
        ctx->launches += per;
        ACP_CUDA(cudaMemcpyAsync(&hs, st, sizeof(QrState), cudaMemcpyDeviceToHost, ctx->stream));
        ACP_CUDA(cudaStreamSynchronize(ctx->stream));
        if (hs.stop) break;
    }
    cudaGraphExecDestroy(exec);
    cudaGraphDestroy(graph);
    ACP_REQUIRE(hs.stop, "QRCP did not terminate");
    const int N = hs.n_mu;
    ACP_REQUIRE(N >= 1, "QRCP selected no rows (zero sketch)");
    if (N > n_mu_max)
        throw Error(ACP_ERR_INVALID, "N_mu = " + std::to_string(N) + " exceeds n_mu_max = " + std::to_string(n_mu_max));
    // Xi
    double* T = ctx->wsd("qr_T", (size_t)N * (Ng - N > 0 ? Ng - N : 1));
    if (Ng > N) {
        k_trsm_cols<<<cdiv(Ng - N, 64), 64, 0, ctx->stream>>>(m, Ng, N, A, T);
        launched(ctx);
    }
    k_scatter_xi<<<dim3(cdiv(Ng, 256), N), 256, 0, ctx->stream>>>(Ng, N, perm, T, Xi, S);
    launched(ctx);
    return N;
}

}  // namespace acp
