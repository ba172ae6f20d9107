// dyson.cu -- Alg. 4 with the SMW update of Eq. dyson4
// and the dynamical matrix of Eqs. SecDeriv/chiterm.
//
//   U~^{k+1} = B + W^k (I - Pi^T v W^k)^{-1} Pi^T v B ,  v B = G   =>
//   Y^k = (I - (K W^k)(S^k,:))^{-1} G(S^k,:),  U^{k+1} = W^k Y^k,  G'^{k+1} = G + (K W^k) Y^k.
// B = v^{-1} G is never formed (it cancels in U = U~ - B).
#include "gemm.cuh"

#include <cmath>
#include <string>
#include <vector>

namespace acp {

// A = I - KW(S, :)  (N x N),  Y = G(S, :)  (N x n)
__global__ void k_smw_gather(int Ng, int N, int n, const int* __restrict__ S, const double* __restrict__ KW,
                             const double* __restrict__ G, double* __restrict__ A, double* __restrict__ Y) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;  // row mu
    const int j = blockIdx.y;                             // column
    if (i >= N) return;
    const int si = S[i];
    if (j < N) A[(size_t)j * N + i] = (i == j ? 1.0 : 0.0) - KW[(size_t)j * Ng + si];
    if (j < n) Y[(size_t)j * N + i] = G[(size_t)j * Ng + si];
}

__global__ void k_diff_norm2(size_t tot, const double* __restrict__ a, const double* __restrict__ b,
                             double* __restrict__ part) {
    __shared__ double red[32];
    double s = 0.0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (size_t)gridDim.x * blockDim.x) {
        const double d = a[i] - b[i];
        s += d * d;
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        part[blockIdx.x] = t;
    }
}

static double diff_norm(acp_context* ctx, const double* a, const double* b, size_t tot) {
    const int blocks = 256;
    double* part = ctx->wsd("diff_part", blocks);
    k_diff_norm2<<<blocks, 256, 0, ctx->stream>>>(tot, a, b, part);
    launched(ctx);
    std::vector<double> h(blocks);
    ACP_CUDA(cudaMemcpyAsync(h.data(), part, blocks * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    ACP_CUDA(cudaStreamSynchronize(ctx->stream));
    double s = 0.0;
    for (double x : h) s += x;
    return std::sqrt(s);
}

// Eq. dyson4 given W (N_g x N) and S:  Y = (I - (K W)(S,:))^{-1} G(S,:),  U = W Y,  Gp = G + (K W) Y.
void smw_update(acp_context* ctx, const double* G, const int* S, const double* W, int N, double* U, double* Gp) {
    const int Ng = ctx->Ng;
    const int n = ctx->dim * ctx->sys.n_atoms;
    double* KW = ctx->wsd("dy_KW", (size_t)Ng * N);
    double* AB = ctx->wsd("dy_AB", (size_t)N * (N + n));  // [A | Y], ld N (blocked LU operand)
    double* A = AB;
    double* Y = AB + (size_t)N * N;
    double* mK = ctx->wsd("dy_multK", Ng);
    copy_cols(ctx, mK, multiplier(ctx, MULT_YUKAWA, 0.0), Ng);
    FopArgs f;
    f.X = W;
    f.Y = KW;
    f.n = N;
    f.mult = mK;
    fourier_op(ctx, f);
    k_smw_gather<<<dim3(cdiv(N, 128), N > n ? N : n), 128, 0, ctx->stream>>>(Ng, N, n, S, KW, G, A, Y);
    launched(ctx);
    // blocked multi-kernel LU (the one-CTA LU measured 13.30 vs 11.71 ms/step on configs[1]: one SM
    // does the O(N^3) work)
    lu_solve_blocked(ctx, AB, N, n);
    gemm_nn(ctx, Ng, N, n, 1.0, W, Ng, Y, N, 0.0, U, Ng);
    if (Gp) {
        copy_cols(ctx, Gp, G, (size_t)Ng * n);
        gemm_nn(ctx, Ng, N, n, 1.0, KW, Ng, Y, N, 1.0, Gp, Ng);
    }
}

void dyson(acp_context* ctx, const double* Psi, const double* eps, const double* V, const double* G,
           const acp_dyson_opts& o, const double* h_theta, const int* h_nu, double* U, double* h_info) {
    const int Ng = ctx->Ng;
    const int n = ctx->dim * ctx->sys.n_atoms;
    const int n_occ = ctx->sys.n_occ;
    ACP_REQUIRE(o.n_outer >= 1 && o.n_cheb >= 1 && o.r_half >= 1, "invalid dyson options");
    const int m = n_occ * 2 * o.r_half;
    const int nmu_max = m < Ng ? m : Ng;
    double* Gp = ctx->wsd("dy_Gp", (size_t)Ng * n);
    double* Uprev = ctx->wsd("dy_Uprev", (size_t)Ng * n);
    int* S = ctx->wsi("dy_S", nmu_max);
    double* Xi = ctx->wsd("dy_Xi", (size_t)Ng * nmu_max);
    double* W = ctx->wsd("dy_W", (size_t)Ng * nmu_max);
    copy_cols(ctx, Gp, G, (size_t)Ng * n);
    fill(ctx, Uprev, (size_t)Ng * n, 0.0);
    // Checks deferred to the end (one host synchronisation per outer iteration: N_mu)
    const int nst = 8 + 2 * o.n_outer;
    long long* dstats = reinterpret_cast<long long*>(ctx->ws("dy_stats", nst * sizeof(long long)));
    double* dpart = ctx->wsd("dy_dn_part", (size_t)o.n_outer * 256);
    ACP_CUDA(cudaMemsetAsync(dstats, 0, nst * sizeof(long long), ctx->stream));
    std::vector<int> Ns(o.n_outer);
    struct DeferGuard {
        acp_context* c;
        ~DeferGuard() { c->defer = 0; }
    } guard{ctx};
    ctx->defer = getenv("ACP_DYSON_SYNC") ? 0 : 1;
    ctx->defer_stats = dstats;
    long long total_solves = 0, total_it = 0;
    int max_it = 0;
    double max_res = 0.0;
    std::vector<double> dn_sync(o.n_outer, 0.0), it_sync(o.n_outer, 0.0);
    // ACP_DYSON_PROF: CUDA events around compress / apply_chi0 / SMW of every outer iteration
    // (printed to stderr at the end; diagnostics only)
    static const bool prof = getenv("ACP_DYSON_PROF") != nullptr;
    std::vector<cudaEvent_t> evs;
    auto mark = [&]() {
        if (!prof) return;
        cudaEvent_t e;
        ACP_CUDA(cudaEventCreate(&e));
        ACP_CUDA(cudaEventRecord(e, ctx->stream));
        evs.push_back(e);
    };
    mark();
    for (int k = 0; k < o.n_outer; ++k) {
        const int N = compress(ctx, Psi, Gp, n, h_theta + (size_t)k * n, h_nu + (size_t)k * o.r_half, o.r_half,
                               o.id_eps, o.n_mu_fixed, nmu_max, S, Xi);
        Ns[k] = N;
        ctx->defer_iter = k;
        mark();
        PcgStats st;
        apply_chi0(ctx, Psi, eps, V, S, Xi, N, 0, N, o.n_cheb, o.cg_tol, o.max_cg_iter, W, &st);
        mark();
        smw_update(ctx, G, S, W, N, U, Gp);
        mark();
        if (ctx->defer) {
            k_diff_norm2<<<256, 256, 0, ctx->stream>>>((size_t)Ng * n, U, Uprev, dpart + (size_t)k * 256);
            launched(ctx);
        } else {
            dn_sync[k] = diff_norm(ctx, U, Uprev, (size_t)Ng * n);
            total_solves += st.n_solved;
            total_it += st.total_iter;
            if (st.max_iter > max_it) max_it = st.max_iter;
            if (st.max_rel_res > max_res) max_res = st.max_rel_res;
            it_sync[k] = (double)st.total_iter;
        }
        copy_cols(ctx, Uprev, U, (size_t)Ng * n);
    }
    std::vector<double> dn(o.n_outer), itk(o.n_outer);
    if (prof) {
        ACP_CUDA(cudaEventSynchronize(evs.back()));
        fprintf(stderr, "[dyson ms: compress / chi0 / smw per outer]");
        for (size_t q = 1; q < evs.size(); ++q) {
            float ms = 0.f;
            ACP_CUDA(cudaEventElapsedTime(&ms, evs[q - 1], evs[q]));
            fprintf(stderr, " %.1f", ms);
        }
        fprintf(stderr, "\n");
        for (auto e : evs) cudaEventDestroy(e);
    }
    if (ctx->defer) {
        std::vector<long long> hs(nst);
        std::vector<double> hp((size_t)o.n_outer * 256);
        ACP_CUDA(cudaMemcpyAsync(hs.data(), dstats, nst * sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
        ACP_CUDA(cudaMemcpyAsync(hp.data(), dpart, hp.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        sync(ctx);
        ctx->defer = 0;
        ctx->launches += hs[3];
        if (hs[6] != 0) throw Error(ACP_ERR_SINGULAR, "singular SMW core in blocked LU");
        if (hs[4] != 0)
            throw Error(ACP_ERR_NOT_CONVERGED,
                        "Sternheimer PCG did not converge in " + std::to_string(o.max_cg_iter) + " iterations");
        total_solves = hs[0];
        total_it = hs[1];
        max_it = (int)hs[2];
        max_res = __builtin_bit_cast(double, hs[5]);
        for (int k = 0; k < o.n_outer; ++k) {
            double s2 = 0.0;
            for (int b = 0; b < 256; ++b) s2 += hp[(size_t)k * 256 + b];  // same order as diff_norm
            dn[k] = std::sqrt(s2);
            itk[k] = (double)hs[8 + 2 * k];
        }
    } else {
        sync(ctx);
        dn = dn_sync;
        itk = it_sync;
    }
    if (h_info) {
        h_info[0] = (double)total_solves;
        h_info[1] = (double)total_it;
        h_info[2] = max_it;
        h_info[3] = max_res;
        for (int k = 0; k < o.n_outer; ++k) {
            h_info[8 + 3 * k] = Ns[k];
            h_info[8 + 3 * k + 1] = dn[k];
            h_info[8 + 3 * k + 2] = itk[k];
        }
    }
}

// ---- dynamical matrix ------------------------------------------------------
// Bin frequency integer (numpy fftfreq order) and the phase e^{-i k.R} of bin (i0, i1).
__device__ __forceinline__ int dm_freq(int i, int N) { return (i < (N + 1) / 2) ? i : i - N; }

// D_loc(I; a, b) = dV sum_r rho(r) d2V_I/dR_a dR_b (r) = (1/N) sum_k Re( h^_I^{ab}(k) conj(rho~(k)) ),
// h^_I^{ab} = (-i k_a)(-i k_b) Khat mhat e^{-i k.R_I}  (Eq. SecDeriv second term).
// One CTA per (I, a, b); dloc[(I d + a) d + b].
__global__ void k_dloc(int n0, int n1, int dim, double L0, double L1, const double* __restrict__ khat,
                       const double* __restrict__ k2, const double* __restrict__ kodd0,
                       const double* __restrict__ kodd1, double Z, double sigma, const double* __restrict__ R,
                       const double2* __restrict__ rhot, double* __restrict__ dloc) {
    __shared__ double red[32];
    const int I = blockIdx.x, a = blockIdx.y / dim, b = blockIdx.y % dim;
    const int N = n0 * n1;
    double s = 0.0;
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        const int i0 = i / n1, i1 = i - i0 * n1;
        const double mh = -Z * exp(-0.5 * sigma * sigma * k2[i]);
        const double ka = a == 0 ? kodd0[i0] : kodd1[i1];
        const double kb = b == 0 ? kodd0[i0] : kodd1[i1];
        const double amp = -ka * kb * khat[i] * mh;
        double t = (double)dm_freq(i0, n0) * R[I * dim] / L0;
        if (dim == 2) t += (double)dm_freq(i1, n1) * R[I * dim + 1] / L1;
        t -= rint(t);
        double sn, cs;
        sincospi(-2.0 * t, &sn, &cs);
        // Re( amp (cs + i sn) * conj(rho) ) = amp (cs rho.x + sn rho.y)
        const double2 r = rhot[i];
        s += amp * (cs * r.x + sn * r.y);
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        dloc[((size_t)I * dim + a) * dim + b] = t / (double)N;
    }
}

// Ion-ion pair Hessian (reading R4): for I != J,
// hpair[((I NA + J) d + a) d + b] = phi''_ab(R_I - R_J) = -(1/Omega) sum_k Khat mhat^2 k_a k_b cos(k.d).
__global__ void k_eii_pairs(int n0, int n1, int dim, double L0, double L1, double Omega,
                            const double* __restrict__ khat, const double* __restrict__ kax0,
                            const double* __restrict__ kax1, const double* __restrict__ k2, double Z,
                            double sigma, const double* __restrict__ R, int NA, double* __restrict__ hpair) {
    __shared__ double red[3][32];
    const int I = blockIdx.x, J = blockIdx.y;
    const int nc = dim == 2 ? 3 : 1;
    double* out = hpair + ((size_t)I * NA + J) * dim * dim;
    if (I == J) {
        if (threadIdx.x < dim * dim) out[threadIdx.x] = 0.0;
        return;
    }
    const int N = n0 * n1;
    const double dx = R[I * dim] - R[J * dim];
    const double dy = dim == 2 ? R[I * dim + 1] - R[J * dim + 1] : 0.0;
    double s[3] = {0.0, 0.0, 0.0};
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        const int i0 = i / n1, i1 = i - i0 * n1;
        const double mh2 = Z * Z * exp(-sigma * sigma * k2[i]);
        double t = (double)dm_freq(i0, n0) * dx / L0;
        if (dim == 2) t += (double)dm_freq(i1, n1) * dy / L1;
        t -= rint(t);
        const double w = khat[i] * mh2 * cospi(2.0 * t);
        const double kx = kax0[i0];
        if (dim == 1) {
            s[0] += w * kx * kx;
        } else {
            const double ky = kax1[i1];
            s[0] += w * kx * kx;
            s[1] += w * kx * ky;
            s[2] += w * ky * ky;
        }
    }
    for (int q = 0; q < nc; ++q) {
        for (int o = 16; o > 0; o >>= 1) s[q] += __shfl_xor_sync(0xffffffffu, s[q], o);
        if ((threadIdx.x & 31) == 0) red[q][threadIdx.x >> 5] = s[q];
    }
    __syncthreads();
    if (threadIdx.x < nc) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[threadIdx.x][w];
        t = -t / Omega;
        if (dim == 1) out[0] = t;
        else if (threadIdx.x == 0) out[0] = t;
        else if (threadIdx.x == 1) { out[1] = t; out[2] = t; }
        else out[3] = t;
    }
}

// D = D_chi + D_loc + D_II (Eq. SecDeriv), mass-scaled and symmetrised; index (I, a) -> I d + a.
// D_II[(I,a),(J,b)] = -phi''_ab(R_I - R_J) (I != J);  D_II[(I,a),(I,b)] = sum_{K != I} phi''_ab(R_I - R_K).
__global__ void k_assemble_D(int NA, int dim, const double* __restrict__ Dchi, const double* __restrict__ dloc,
                             const double* __restrict__ hpair, const double* __restrict__ mass,
                             double* __restrict__ D) {
    const int n = NA * dim;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;  // row (I, a)
    const int q = blockIdx.y;                             // column (J, b)
    if (p >= n) return;
    auto entry = [&](int r, int c) {
        const int I = r / dim, a = r % dim, J = c / dim, b = c % dim;
        double v = Dchi[(size_t)c * n + r];
        if (I == J) {
            v += dloc[((size_t)I * dim + a) * dim + b];
            double s = 0.0;
            for (int K = 0; K < NA; ++K) s += hpair[(((size_t)I * NA + K) * dim + a) * dim + b];
            v += s;
        } else {
            v -= hpair[(((size_t)I * NA + J) * dim + a) * dim + b];
        }
        return v;
    };
    const double v = 0.5 * (entry(p, q) + entry(q, p));
    const double mm = mass ? sqrt(mass[p / dim] * mass[q / dim]) : 1.0;
    D[(size_t)q * n + p] = v / mm;
}

void dynamical_matrix(acp_context* ctx, const double* h_R, const double* rho, const double* G, const double* U,
                      const double* h_masses, double* h_D, double* h_lambda) {
    const int Ng = ctx->Ng;
    const int NA = ctx->sys.n_atoms;
    const int dim = ctx->dim;
    const int n = dim * NA;
    double* dR = ctx->wsd("dm_R", (size_t)NA * dim);
    ACP_CUDA(cudaMemcpyAsync(dR, h_R, (size_t)NA * dim * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    double* dm = nullptr;
    if (h_masses) {
        dm = ctx->wsd("dm_mass", NA);
        ACP_CUDA(cudaMemcpyAsync(dm, h_masses, NA * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    }
    double* Dchi = ctx->wsd("dm_Dchi", (size_t)n * n);
    gemm_tn(ctx, Ng, n, n, ctx->dV, G, Ng, U, Ng, Dchi);
    double2* rhot = static_cast<double2*>(ctx->ws("dm_rhot", (size_t)Ng * sizeof(double2)));
    real_spectrum(ctx, rho, rhot);
    double* dloc = ctx->wsd("dm_dloc", (size_t)NA * dim * dim);
    const double* kodd1 = dim == 2 ? ctx->d_kaxodd[1] : ctx->d_kaxodd[0];
    const double* kax1 = dim == 2 ? ctx->d_kax[1] : ctx->d_kax[0];
    k_dloc<<<dim3(NA, dim * dim), 256, 0, ctx->stream>>>(ctx->n[0], ctx->n[1], dim, ctx->sys.cell[0],
                                                          ctx->sys.cell[1], ctx->d_khat, ctx->d_k2,
                                                          ctx->d_kaxodd[0], kodd1, ctx->sys.Z, ctx->sys.sigma, dR,
                                                          rhot, dloc);
    launched(ctx);
    double* hpair = ctx->wsd("dm_hpair", (size_t)NA * NA * dim * dim);
    k_eii_pairs<<<dim3(NA, NA), 256, 0, ctx->stream>>>(ctx->n[0], ctx->n[1], dim, ctx->sys.cell[0],
                                                        ctx->sys.cell[1], ctx->Omega, ctx->d_khat, ctx->d_kax[0],
                                                        kax1, ctx->d_k2, ctx->sys.Z, ctx->sys.sigma, dR, NA, hpair);
    launched(ctx);
    double* D = ctx->wsd("dm_D", (size_t)n * n);
    k_assemble_D<<<dim3(cdiv(n, 128), n), 128, 0, ctx->stream>>>(NA, dim, Dchi, dloc, hpair, dm, D);
    launched(ctx);
    ACP_CUDA(cudaMemcpyAsync(h_D, D, (size_t)n * n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    if (h_lambda) {
        double* Dw = ctx->wsd("dm_Dwork", (size_t)n * n);
        double* w = ctx->wsd("dm_w", n);
        copy_cols(ctx, Dw, D, (size_t)n * n);
        sym_eig(ctx, Dw, n, w, nullptr);
        ACP_CUDA(cudaMemcpyAsync(h_lambda, w, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    }
    sync(ctx);
}

void perturbations(acp_context* ctx, const double* h_R, double* G) {
    const int NA = ctx->sys.n_atoms;
    const int n = ctx->dim * NA;
    double* dR = ctx->wsd("pt_R", (size_t)NA * ctx->dim);  // N_A x d row-major
    ACP_CUDA(cudaMemcpyAsync(dR, h_R, (size_t)NA * ctx->dim * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    double2* spec = static_cast<double2*>(ctx->ws("pt_spec", (size_t)ctx->Ng * n * sizeof(double2)));
    spectrum_G(ctx, dR, spec);
    ifft_hermitian(ctx, spec, n, G);
    sync(ctx);
}

}  // namespace acp
