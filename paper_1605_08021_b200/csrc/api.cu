// api.cu -- extern "C" entry points of include/acp_b200.h.  Argument checking,
// device selection and error translation only; all arithmetic lives in the kernels.
#include <mutex>
#include <map>
#include "common.cuh"

#include <cmath>

namespace acp {
void func_attr(const void* fn, size_t smem, bool nonportable_cluster) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, std::pair<size_t, bool>> done;
    int dev = 0;
    ACP_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    auto& d = done[{dev, fn}];
    if (d.first < smem) {
        ACP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        d.first = smem;
    }
    if (nonportable_cluster && !d.second) {
        ACP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        d.second = true;
    }
}
}  // namespace acp


using acp::Error;

namespace {

int fail(acp_context* ctx, int code, const std::string& msg) {
    if (ctx) ctx->err = msg;
    return code;
}

template <class F>
int guarded(acp_context* ctx, F&& f) {
    if (!ctx) return ACP_ERR_INVALID;
    try {
        ACP_CUDA(cudaSetDevice(ctx->device));
        f();
        return ACP_OK;
    } catch (const Error& e) {
        return fail(ctx, e.code, e.what());
    } catch (const std::exception& e) {
        return fail(ctx, ACP_ERR_CUDA, e.what());
    }
}

}  // namespace

extern "C" {

const char* acp_version(void) { return "acp_b200 1.0 sm_100a fp64"; }

int acp_create(const acp_system* sys, int device, acp_context** out) {
    if (!sys || !out) return ACP_ERR_INVALID;
    *out = nullptr;
    if (sys->dim != 1 && sys->dim != 2) return ACP_ERR_INVALID;
    if (sys->grid[0] < 4 || sys->n_atoms < 1 || sys->n_occ < 1 || sys->cell[0] <= 0 || sys->kappa <= 0 ||
        sys->eps0 <= 0 || sys->sigma <= 0 || sys->occ <= 0)
        return ACP_ERR_INVALID;
    if (sys->dim == 2 && (sys->grid[1] < 4 || sys->cell[1] <= 0)) return ACP_ERR_INVALID;
    const long long ng = (long long)sys->grid[0] * (sys->dim == 2 ? sys->grid[1] : 1);
    if (sys->n_occ >= ng || ng > (1LL << 24)) return ACP_ERR_INVALID;
    acp_context* ctx = new acp_context();
    ctx->sys = *sys;
    ctx->device = device;
    ctx->dim = sys->dim;
    ctx->Ng = (int)ng;
    ctx->Omega = sys->cell[0] * (sys->dim == 2 ? sys->cell[1] : 1.0);
    ctx->dV = ctx->Omega / ctx->Ng;
    try {
        ACP_CUDA(cudaSetDevice(device));
        ACP_CUDA(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
        ctx->stream = ctx->own_stream;
        ACP_CUDA(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
        for (int g = 1; g < acp::PCG_MAXG; ++g) {
            ACP_CUDA(cudaStreamCreateWithFlags(&ctx->gstream[g], cudaStreamNonBlocking));
            ACP_CUDA(cudaEventCreateWithFlags(&ctx->ev_join[g], cudaEventDisableTiming));
        }
        ACP_CUDA(cudaMallocHost(&ctx->pinned, 4096));
        acp::fft_init(ctx);
    } catch (const Error& e) {
        int code = e.code;
        acp_destroy(ctx);
        return code;
    } catch (const std::exception&) {
        acp_destroy(ctx);
        return ACP_ERR_CUDA;
    }
    *out = ctx;
    return ACP_OK;
}

int acp_destroy(acp_context* ctx) {
    if (!ctx) return ACP_OK;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    for (auto& kv : ctx->graphs)
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    for (auto& kv : ctx->bufs)
        if (kv.second.ptr) cudaFree(kv.second.ptr);
    acp::fft_free(ctx);
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    for (int g = 1; g < acp::PCG_MAXG; ++g) {
        if (ctx->gstream[g]) {
            cudaStreamSynchronize(ctx->gstream[g]);
            cudaStreamDestroy(ctx->gstream[g]);
        }
        if (ctx->ev_join[g]) cudaEventDestroy(ctx->ev_join[g]);
    }
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx;
    return ACP_OK;
}

const char* acp_last_error(const acp_context* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int acp_set_stream(acp_context* ctx, void* s) {
    if (!ctx) return ACP_ERR_INVALID;
    ctx->stream = s ? static_cast<cudaStream_t>(s) : ctx->own_stream;
    return ACP_OK;
}

long long acp_kernel_launches(const acp_context* ctx) { return ctx ? ctx->launches : 0; }

int acp_ground_state(acp_context* ctx, const double* h_R, const acp_scf_opts* opts, double* d_Psi, double* d_eps,
                     double* d_rho, double* d_V, double* d_G, double* h_info) {
    if (!ctx || !h_R || !opts || !d_Psi || !d_eps || !d_rho || !d_V) return ACP_ERR_INVALID;
    return guarded(ctx, [&] { acp::ground_state(ctx, h_R, *opts, d_Psi, d_eps, d_rho, d_V, d_G, h_info); });
}

int acp_perturbations(acp_context* ctx, const double* h_R, double* d_G) {
    if (!ctx || !h_R || !d_G) return ACP_ERR_INVALID;
    return guarded(ctx, [&] { acp::perturbations(ctx, h_R, d_G); });
}

int acp_compress(acp_context* ctx, const double* d_Psi, const double* d_Gp, int n_cols, const double* h_theta,
                 const int* h_nu, int r_half, double id_eps, int n_mu_fixed, int n_mu_max, int* d_S, double* d_Xi,
                 int* h_n_mu) {
    if (!ctx || !d_Psi || !d_Gp || !h_theta || !h_nu || !d_S || !d_Xi || !h_n_mu) return ACP_ERR_INVALID;
    if (n_cols < 1 || r_half < 1 || r_half > n_cols || n_mu_max < 1) return fail(ctx, ACP_ERR_INVALID, "bad sizes");
    for (int q = 0; q < r_half; ++q)
        if (h_nu[q] < 1 || h_nu[q] > n_cols) return fail(ctx, ACP_ERR_INVALID, "nu out of range 1..n_cols");
    return guarded(ctx, [&] {
        *h_n_mu = acp::compress(ctx, d_Psi, d_Gp, n_cols, h_theta, h_nu, r_half, id_eps, n_mu_fixed, n_mu_max, d_S,
                                d_Xi);
        acp::sync(ctx);
    });
}

int acp_qrs_begin(acp_context* ctx, const double* d_Psi, const double* d_Gp, int n_cols, const double* h_theta,
                  const int* h_nu, int r_half, int col_begin, int col_end, int n_mu_fixed, int n_mu_max,
                  int* h_m) {
    if (!ctx || !d_Psi || !d_Gp || !h_theta || !h_nu || !h_m) return ACP_ERR_INVALID;
    if (n_cols < 1 || r_half < 1 || r_half > n_cols || n_mu_max < 1) return fail(ctx, ACP_ERR_INVALID, "bad sizes");
    if (col_begin < 0 || col_end < col_begin || col_end > ctx->Ng) return fail(ctx, ACP_ERR_INVALID, "bad column range");
    for (int q = 0; q < r_half; ++q)
        if (h_nu[q] < 1 || h_nu[q] > n_cols) return fail(ctx, ACP_ERR_INVALID, "nu out of range 1..n_cols");
    return guarded(ctx, [&] {
        *h_m = acp::qrs_begin(ctx, d_Psi, d_Gp, n_cols, h_theta, h_nu, r_half, col_begin, col_end, n_mu_fixed,
                              n_mu_max);
    });
}

int acp_qrs_step(acp_context* ctx, int s, const double* d_recv, int world, double id_eps, double* d_send) {
    if (!ctx || !d_recv || !d_send || world < 1 || s < 0) return ACP_ERR_INVALID;
    if (ctx->qrs_m <= 0) return fail(ctx, ACP_ERR_INVALID, "acp_qrs_step before acp_qrs_begin");
    return guarded(ctx, [&] { acp::qrs_step(ctx, s, d_recv, world, id_eps, d_send); });
}

int acp_qrs_status(acp_context* ctx, int* h_stopped, int* h_n_mu) {
    if (!ctx || !h_stopped || !h_n_mu) return ACP_ERR_INVALID;
    if (ctx->qrs_m <= 0) return fail(ctx, ACP_ERR_INVALID, "acp_qrs_status before acp_qrs_begin");
    return guarded(ctx, [&] { acp::qrs_status(ctx, h_stopped, h_n_mu); });
}

int acp_qrs_finish(acp_context* ctx, int* d_S, double* d_XiT, int* h_n_mu) {
    if (!ctx || !d_S || !d_XiT || !h_n_mu) return ACP_ERR_INVALID;
    if (ctx->qrs_m <= 0) return fail(ctx, ACP_ERR_INVALID, "acp_qrs_finish before acp_qrs_begin");
    return guarded(ctx, [&] {
        *h_n_mu = acp::qrs_finish(ctx, d_S, d_XiT);
        acp::sync(ctx);
    });
}

int acp_apply_chi0(acp_context* ctx, const double* d_Psi, const double* d_eps, const double* d_V, const int* d_S,
                   const double* d_Xi, int n_mu, int mu_begin, int mu_end, int n_cheb, double cg_tol, int max_iter,
                   double* d_W, double* h_info) {
    if (!ctx || !d_Psi || !d_eps || !d_V || !d_S || !d_Xi || !d_W) return ACP_ERR_INVALID;
    if (n_mu < 1 || mu_begin < 0 || mu_end > n_mu || mu_begin > mu_end || n_cheb < 1 || cg_tol <= 0 ||
        max_iter < 1)
        return fail(ctx, ACP_ERR_INVALID, "bad sizes");
    return guarded(ctx, [&] {
        acp::PcgStats st;
        acp::apply_chi0(ctx, d_Psi, d_eps, d_V, d_S, d_Xi, n_mu, mu_begin, mu_end, n_cheb, cg_tol, max_iter, d_W,
                        &st);
        acp::sync(ctx);
        if (h_info) {
            h_info[0] = st.max_iter;
            h_info[1] = (double)st.total_iter;
            h_info[2] = st.max_rel_res;
            h_info[3] = st.n_solved;
        }
    });
}

int acp_dyson(acp_context* ctx, const double* d_Psi, const double* d_eps, const double* d_V, const double* d_G,
              const acp_dyson_opts* opts, const double* h_theta, const int* h_nu, double* d_U, double* h_info) {
    if (!ctx || !d_Psi || !d_eps || !d_V || !d_G || !opts || !h_theta || !h_nu || !d_U) return ACP_ERR_INVALID;
    return guarded(ctx, [&] { acp::dyson(ctx, d_Psi, d_eps, d_V, d_G, *opts, h_theta, h_nu, d_U, h_info); });
}

int acp_smw_update(acp_context* ctx, const double* d_G, const int* d_S, const double* d_W, int n_mu, double* d_U,
                   double* d_Gp) {
    if (!ctx || !d_G || !d_S || !d_W || !d_U || n_mu < 1) return ACP_ERR_INVALID;
    return guarded(ctx, [&] {
        acp::smw_update(ctx, d_G, d_S, d_W, n_mu, d_U, d_Gp);
        acp::sync(ctx);
    });
}

int acp_dynamical_matrix(acp_context* ctx, const double* h_R, const double* d_rho, const double* d_G,
                         const double* d_U, const double* h_masses, double* h_D, double* h_lambda) {
    if (!ctx || !h_R || !d_rho || !d_G || !d_U || !h_D) return ACP_ERR_INVALID;
    return guarded(ctx, [&] { acp::dynamical_matrix(ctx, h_R, d_rho, d_G, d_U, h_masses, h_D, h_lambda); });
}

int acp_fourier_apply(acp_context* ctx, const double* d_X, int n, int which_mult, double tau, const double* d_diag,
                      const double* d_shift, double* d_Y) {
    if (!ctx || !d_X || !d_Y || n < 0 || which_mult < 0 || which_mult > 3) return ACP_ERR_INVALID;
    return guarded(ctx, [&] {
        acp::FopArgs f;
        f.X = d_X;
        f.Y = d_Y;
        f.n = n;
        f.mult = acp::multiplier(ctx, (acp::MultKind)which_mult, tau);
        f.diag = d_diag;
        f.shift = d_shift;
        acp::fourier_op(ctx, f);
        acp::sync(ctx);
    });
}

int acp_gemm_tn(acp_context* ctx, int K, int m, int n, double alpha, const double* d_A, int lda, const double* d_B,
                int ldb, double* d_C) {
    if (!ctx || !d_A || !d_B || !d_C || K < 1 || m < 0 || n < 0 || lda < K || ldb < K) return ACP_ERR_INVALID;
    return guarded(ctx, [&] {
        acp::gemm_tn(ctx, K, m, n, alpha, d_A, lda, d_B, ldb, d_C);
        acp::sync(ctx);
    });
}

int acp_gemm_nn(acp_context* ctx, int M, int K, int n, double alpha, const double* d_A, int lda, const double* d_B,
                int ldb, double beta, double* d_C, int ldc) {
    if (!ctx || !d_A || !d_B || !d_C || M < 0 || K < 1 || n < 0 || lda < M || ldb < K || ldc < M)
        return ACP_ERR_INVALID;
    return guarded(ctx, [&] {
        acp::gemm_nn(ctx, M, K, n, alpha, d_A, lda, d_B, ldb, beta, d_C, ldc);
        acp::sync(ctx);
    });
}

int acp_lu_solve(acp_context* ctx, int n, int nrhs, double* d_A, double* d_B) {
    if (!ctx || !d_A || (nrhs > 0 && !d_B) || n < 1 || nrhs < 0) return ACP_ERR_INVALID;
    return guarded(ctx, [&] {
        double* AB = ctx->wsd("api_luAB", (size_t)n * (n + nrhs));
        ACP_CUDA(cudaMemcpyAsync(AB, d_A, (size_t)n * n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
        if (nrhs)
            ACP_CUDA(cudaMemcpyAsync(AB + (size_t)n * n, d_B, (size_t)n * nrhs * sizeof(double),
                                     cudaMemcpyDeviceToDevice, ctx->stream));
        acp::lu_solve_blocked(ctx, AB, n, nrhs);
        ACP_CUDA(cudaMemcpyAsync(d_A, AB, (size_t)n * n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
        if (nrhs)
            ACP_CUDA(cudaMemcpyAsync(d_B, AB + (size_t)n * n, (size_t)n * nrhs * sizeof(double),
                                     cudaMemcpyDeviceToDevice, ctx->stream));
        acp::sync(ctx);
    });
}

int acp_sym_eigvals(acp_context* ctx, int n, const double* d_A, double* d_w) {
    if (!ctx || !d_A || !d_w || n < 1) return ACP_ERR_INVALID;
    return guarded(ctx, [&] {
        double* Aw = ctx->wsd("api_eigA", (size_t)n * n);
        ACP_CUDA(cudaMemcpyAsync(Aw, d_A, (size_t)n * n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
        acp::sym_eig(ctx, Aw, n, d_w, nullptr);
        acp::sync(ctx);
    });
}

int acp_kernel_bench(acp_context* ctx, int which, const double* d_Psi, const double* d_V, const double* d_X,
                     int n_cols, double* d_Y, int reps) {
    if (!ctx || !d_Psi || !d_V || !d_X || !d_Y || n_cols < 1 || reps < 1 || which < 0 || which > 4)
        return ACP_ERR_INVALID;
    return guarded(ctx, [&] { acp::kernel_bench(ctx, which, d_Psi, d_V, d_X, n_cols, d_Y, reps); });
}

void* acp_get_stream(const acp_context* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

}  // extern "C"
