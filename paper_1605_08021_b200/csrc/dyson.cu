// dyson.cu -- Alg. 4 with the SMW update of Eq. dyson4
// and the dynamical matrix of Eqs. SecDeriv/chiterm.
//
//   U~^{k+1} = B + W^k (I - Pi^T v W^k)^{-1} Pi^T v B ,  v B = G   =>
//   Y^k = (I - (K W^k)(S^k,:))^{-1} G(S^k,:),  U^{k+1} = W^k Y^k,  G'^{k+1} = G + (K W^k) Y^k.
// B = v^{-1} G is never formed (it cancels in U = U~ - B).
#include "gemm.cuh"

#include <cmath>
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
    double* A = ctx->wsd("dy_A", (size_t)N * N);
    double* Y = ctx->wsd("dy_Y", (size_t)N * n);
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
    lu_solve(ctx, A, N, Y, n);
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
    long long total_solves = 0, total_it = 0;
    int max_it = 0;
    double max_res = 0.0;
    for (int k = 0; k < o.n_outer; ++k) {
        const int N = compress(ctx, Psi, Gp, n, h_theta + (size_t)k * n, h_nu + (size_t)k * o.r_half, o.r_half,
                               o.id_eps, o.n_mu_fixed, nmu_max, S, Xi);
        PcgStats st;
        apply_chi0(ctx, Psi, eps, V, S, Xi, N, 0, N, o.n_cheb, o.cg_tol, o.max_cg_iter, W, &st);
        smw_update(ctx, G, S, W, N, U, Gp);
        const double dn = diff_norm(ctx, U, Uprev, (size_t)Ng * n);
        copy_cols(ctx, Uprev, U, (size_t)Ng * n);
        total_solves += st.n_solved;
        total_it += st.total_iter;
        if (st.max_iter > max_it) max_it = st.max_iter;
        if (st.max_rel_res > max_res) max_res = st.max_rel_res;
        if (h_info) {
            h_info[8 + 3 * k] = N;
            h_info[8 + 3 * k + 1] = dn;
            h_info[8 + 3 * k + 2] = (double)st.total_iter;
        }
    }
    sync(ctx);
    if (h_info) {
        h_info[0] = (double)total_solves;
        h_info[1] = (double)total_it;
        h_info[2] = max_it;
        h_info[3] = max_res;
    }
}

// ---- dynamical matrix ------------------------------------------------------
// D_loc(I; a, b) = dV sum rho d2V_I = (1/N) sum_k Re( h^_I(k) conj(rho~(k)) ),
// h^_I = (-i k_a)(-i k_b) Khat mhat e^{-i k R_I} (1D: a = b = 0).
__global__ void k_dloc(int N, double L, const double* __restrict__ khat, const double* __restrict__ kodd,
                       const double* __restrict__ k2, double Z, double sigma, const double* __restrict__ R,
                       const double2* __restrict__ rhot, double* __restrict__ dloc) {
    __shared__ double red[32];
    const int I = blockIdx.x;
    double s = 0.0;
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        const int m = (i < (N + 1) / 2) ? i : i - N;
        const double mh = -Z * exp(-0.5 * sigma * sigma * k2[i]);
        const double amp = -kodd[i] * kodd[i] * khat[i] * mh;
        double sn, cs;
        sincospi(-2.0 * (double)m * R[I] / L, &sn, &cs);
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
        dloc[I] = t / (double)N;
    }
}

// hpair[I + J NA] = phi''(R_I - R_J) = -(1/Omega) sum_k Khat mhat^2 k^2 cos(k d)   (1D)
__global__ void k_eii_pairs(int N, double L, double Omega, const double* __restrict__ khat,
                            const double* __restrict__ kfull, double Z, double sigma, const double* __restrict__ R,
                            int NA, double* __restrict__ hpair) {
    __shared__ double red[32];
    const int I = blockIdx.x, J = blockIdx.y;
    if (I == J) {
        if (threadIdx.x == 0) hpair[I + J * NA] = 0.0;
        return;
    }
    const double d = R[I] - R[J];
    double s = 0.0;
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        const int m = (i < (N + 1) / 2) ? i : i - N;
        const double k = kfull[i];
        const double mh2 = Z * Z * exp(-sigma * sigma * k * k);
        s += khat[i] * mh2 * k * k * cospi(2.0 * (double)m * d / L);
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        hpair[I + J * NA] = -t / Omega;
    }
}

// D = D_chi + D_loc + D_II, mass-scaled and symmetrised (1D: index I).
__global__ void k_assemble_D(int NA, const double* __restrict__ Dchi, const double* __restrict__ dloc,
                             const double* __restrict__ hpair, const double* __restrict__ mass,
                             double* __restrict__ D) {
    const int I = blockIdx.x * blockDim.x + threadIdx.x;
    const int J = blockIdx.y;
    if (I >= NA) return;
    auto entry = [&](int a, int b) {
        double v = Dchi[(size_t)b * NA + a];
        if (a == b) {
            v += dloc[a];
            double s = 0.0;
            for (int K = 0; K < NA; ++K) s += hpair[a + K * NA];
            v += s;
        } else {
            v -= hpair[a + b * NA];
        }
        return v;
    };
    const double v = 0.5 * (entry(I, J) + entry(J, I));
    const double mm = mass ? sqrt(mass[I] * mass[J]) : 1.0;
    D[(size_t)J * NA + I] = v / mm;
}

void dynamical_matrix(acp_context* ctx, const double* h_R, const double* rho, const double* G, const double* U,
                      const double* h_masses, double* h_D, double* h_lambda) {
    ACP_REQUIRE(ctx->dim == 1, "2D dynamical matrix not built in this round");
    const int Ng = ctx->Ng;
    const int NA = ctx->sys.n_atoms;
    const int n = NA;
    double* dR = ctx->wsd("dm_R", NA);
    ACP_CUDA(cudaMemcpyAsync(dR, h_R, NA * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    double* dm = nullptr;
    if (h_masses) {
        dm = ctx->wsd("dm_mass", NA);
        ACP_CUDA(cudaMemcpyAsync(dm, h_masses, NA * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    }
    double* Dchi = ctx->wsd("dm_Dchi", (size_t)n * n);
    gemm_tn(ctx, Ng, n, n, ctx->dV, G, Ng, U, Ng, Dchi);
    double2* rhot = static_cast<double2*>(ctx->ws("dm_rhot", (size_t)Ng * sizeof(double2)));
    real_spectrum(ctx, rho, rhot);
    double* dloc = ctx->wsd("dm_dloc", NA);
    k_dloc<<<NA, 256, 0, ctx->stream>>>(Ng, ctx->sys.cell[0], ctx->d_khat, ctx->d_kodd, ctx->d_k2, ctx->sys.Z,
                                         ctx->sys.sigma, dR, rhot, dloc);
    launched(ctx);
    double* hpair = ctx->wsd("dm_hpair", (size_t)NA * NA);
    k_eii_pairs<<<dim3(NA, NA), 256, 0, ctx->stream>>>(Ng, ctx->sys.cell[0], ctx->Omega, ctx->d_khat, ctx->d_kfull,
                                                        ctx->sys.Z, ctx->sys.sigma, dR, NA, hpair);
    launched(ctx);
    double* D = ctx->wsd("dm_D", (size_t)n * n);
    k_assemble_D<<<dim3(cdiv(NA, 128), NA), 128, 0, ctx->stream>>>(NA, Dchi, dloc, hpair, dm, D);
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
    double* dR = ctx->wsd("pt_R", (size_t)NA * ctx->dim);
    ACP_CUDA(cudaMemcpyAsync(dR, h_R, (size_t)NA * ctx->dim * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    double2* spec = static_cast<double2*>(ctx->ws("pt_spec", (size_t)ctx->Ng * n * sizeof(double2)));
    spectrum_G(ctx, dR, spec);
    ifft_hermitian(ctx, spec, n, G);
    sync(ctx);
}

}  // namespace acp
