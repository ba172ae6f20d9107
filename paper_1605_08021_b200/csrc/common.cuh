// common.cuh -- shared declarations of the B200 ACP library (internal).
//
// Context, error handling, workspace and launch accounting.  All kernels are
// written for sm_100a (B200); fp64 throughout.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/acp_b200.h"

namespace acp {

constexpr int PCG_MAXG = 8;  // concurrent PCG node groups (streams)

struct Error : public std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define ACP_CUDA(call)                                                                   \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            throw ::acp::Error(ACP_ERR_CUDA, std::string(#call) + ": " +                 \
                                                 cudaGetErrorString(e_) + " @" +         \
                                                 __FILE__ + ":" + std::to_string(__LINE__)); \
    } while (0)

#define ACP_REQUIRE(cond, msg)                                                           \
    do {                                                                                 \
        if (!(cond)) throw ::acp::Error(ACP_ERR_INVALID, std::string(msg));              \
    } while (0)

// FFT plan for one 1D length (Stockham autosort, radices 8/4/2/5/3).
struct FftPlan {
    int N = 0;
    int npass = 0;
    int radix[24] = {0};
    int twoff[25] = {0};  // per-pass twiddle table offsets (entries), twoff[npass] = total
};

// Grow-only device buffer.
struct DevBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
};

}  // namespace acp

struct acp_context {
    acp_system sys{};
    int device = 0;
    int dim = 1;
    int Ng = 0;
    double dV = 0.0, Omega = 0.0;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;
    // PCG node groups 1.. run on gstream[g] (forked from / joined to `stream`)
    cudaStream_t gstream[acp::PCG_MAXG] = {};
    cudaEvent_t ev_fork = nullptr;
    cudaEvent_t ev_join[acp::PCG_MAXG] = {};
    int f2_alt = 0;                       // 2D K1 workspace selector: the group being enqueued
    // Deferred checks (acp_dyson): PCG statistics / convergence, LU status and the iteration
    // differences stay on the device (defer_stats, indexed by defer_iter) and are read once at the
    // end, so an outer iteration has a single host synchronisation (the QRCP rank N_mu).
    int defer = 0;
    int defer_iter = 0;
    long long* defer_stats = nullptr;  // see DeferStats in pcg.cu
    std::string err;
    long long launches = 0;

    // Grid / Fourier tables.  Axis a has n[a] points (n[1] = 1 in 1D); bins in numpy fft order,
    // flattened C order (bin index k0 * n1 + k1).
    int n[2] = {1, 1};
    acp::FftPlan plan;           // axis 0 (1D: the whole grid)
    acp::FftPlan plan1;          // axis 1 (2D only)
    double2* d_tw = nullptr;     // exp(-2 pi i m / n0), m < n0
    double2* d_tw1 = nullptr;    // exp(-2 pi i m / n1) (2D)
    double* d_k2 = nullptr;      // |k|^2 per bin (N_g)
    double* d_khat = nullptr;    // Yukawa symbol 4 pi / (eps0 (|k|^2 + kappa^2)) per bin (N_g)
    double* d_kax[2] = {nullptr, nullptr};     // k_a per axis index (length n[a])
    double* d_kaxodd[2] = {nullptr, nullptr};  // k_a with the Nyquist entry zeroed (odd multipliers)
    double* d_kodd = nullptr;    // alias of d_kaxodd[0] (1D code)
    double* d_kfull = nullptr;   // alias of d_kax[0]
    double* d_mult = nullptr;    // scratch multiplier table (N_g)
    // 2D operator geometry: a cluster of cs CTAs per column pair, r0 = n0/cs rows and
    // c1 = n1/cs columns per CTA; threads per CTA and elements per thread of the FFT engine.
    int cs = 1, r0 = 0, c1 = 0, fthreads = 0, fept = 0;
    size_t fsmem = 0;
    int fnp = 1;                         // 2D: column pairs per cluster for operator launches
    bool pdl = false;                    // launch with programmatic dependent launch (PCG graph)
    int fthreads1 = 0, fept1 = 0;        // 2D: geometry of the one-pair setup transforms
    int fct = 0;                         // 1D: a compiled-length FFT kernel matches the plan
    double2* d_twf2c = nullptr;          // fused 2D operator (fft2c.cu): exp(-2 pi i j / n0), j < n0
    int f2c_maxcl = 0;                   // fused 2D operator: resident CTAs (queried once)
    // sharded QRCP (qrcp.cu, acp_qrs_*): this rank's column block and the factorisation sizes
    int qrs_m = 0, qrs_kmax = 0, qrs_col0 = 0, qrs_nloc = 0, qrs_fixed = 0;
    size_t fsmem1 = 0;

    std::map<std::string, acp::DevBuf> bufs;
    void* pinned = nullptr;  // 4 KiB pinned host scratch for small device->host reads

    // Instantiated CUDA graphs keyed by (kernel sequence, shapes, pointers): re-used across calls.
    struct GraphEntry {
        cudaGraphExec_t exec = nullptr;
        long long launches = 0;
    };
    std::map<std::string, GraphEntry> graphs;

    // Workspace of at least `bytes` bytes under `name` (contents not preserved on growth).
    void* ws(const std::string& name, size_t bytes) {
        acp::DevBuf& b = bufs[name];
        if (b.bytes < bytes) {
            // a cached graph may hold this buffer's old address (and a later allocation may reuse
            // it, so pointer-keyed lookups cannot tell): drop every cached graph on reallocation
            if (b.ptr) {
                cudaDeviceSynchronize();  // both PCG streams
                for (auto& kv : graphs)
                    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
                graphs.clear();
                cudaFree(b.ptr);
            }
            b.ptr = nullptr;
            b.bytes = 0;
            size_t nb = bytes < 256 ? 256 : bytes;
            cudaError_t e = cudaMalloc(&b.ptr, nb);
            if (e != cudaSuccess)
                throw acp::Error(ACP_ERR_ALLOC, "cudaMalloc(" + std::to_string(nb) + ") for " + name +
                                                    ": " + cudaGetErrorString(e));
            b.bytes = nb;
        }
        return b.ptr;
    }
    double* wsd(const std::string& name, size_t n) { return static_cast<double*>(ws(name, n * sizeof(double))); }
    int* wsi(const std::string& name, size_t n) { return static_cast<int*>(ws(name, n * sizeof(int))); }
};

namespace acp {

// Programmatic dependent launch (PDL, sm_90+): kernels of the PCG loop are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, wait for their predecessor's results with
// griddepcontrol.wait (a no-op without the attribute) and let their successor be scheduled early
// with griddepcontrol.launch_dependents.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Record one kernel launch (call right after <<<>>>); checks launch errors.
// Debug knob ACP_SYNC_CHECK=1: synchronise after every launch outside stream capture, so a
// faulting kernel is reported at its own launch site (with ACP_PCG_NOGRAPH=1 for the PCG loop).
#define launched(ctx, ...) launched_at(ctx, __FILE__, __LINE__, ##__VA_ARGS__)
inline void launched_at(acp_context* ctx, const char* file, int line, int n = 1) {
    ctx->launches += n;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        throw Error(ACP_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e) + " @" + file + ":" +
                                      std::to_string(line));
    static const bool chk = getenv("ACP_SYNC_CHECK") != nullptr;
    if (chk) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(ctx->stream, &cs);
        if (cs == cudaStreamCaptureStatusNone) {
            e = cudaStreamSynchronize(ctx->stream);
            if (e != cudaSuccess)
                throw Error(ACP_ERR_CUDA, std::string("kernel execution: ") + cudaGetErrorString(e) + " @" + file +
                                              ":" + std::to_string(line));
        }
    }
}

// Raise a kernel's dynamic shared-memory limit to >= smem bytes (and allow non-portable cluster
// sizes) on the CURRENT device.  Function attributes belong to a device context, so the record
// of what was set is keyed by (device, kernel); it is mutex-protected (api.cu).
void func_attr(const void* fn, size_t smem, bool nonportable_cluster = false);

inline void sync(acp_context* ctx) { ACP_CUDA(cudaStreamSynchronize(ctx->stream)); }

inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

// Capture `body` (a sequence of launches on ctx->stream) into a graph once per key and return
// the instantiated executable.  The key must encode every shape and pointer the launches use.
template <class F>
cudaGraphExec_t graph_cached(acp_context* ctx, const std::string& key, F&& body) {
    auto it = ctx->graphs.find(key);
    if (it != ctx->graphs.end()) return it->second.exec;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t e = nullptr;
    const long long before = ctx->launches;
    ACP_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    try {
        body();
    } catch (...) {
        cudaStreamEndCapture(ctx->stream, &g);
        if (g) cudaGraphDestroy(g);
        throw;
    }
    ACP_CUDA(cudaStreamEndCapture(ctx->stream, &g));
    ACP_CUDA(cudaGraphInstantiate(&e, g, 0));
    cudaGraphDestroy(g);
    auto& ent = ctx->graphs[key];
    ent.exec = e;
    ent.launches = ctx->launches - before;
    ctx->launches = before;
    return e;
}
// Bound the graph cache (each new shape / pointer set adds entries): called where no cached
// executable is held by the caller; waits for the device before destroying.
inline void graph_cache_trim(acp_context* ctx, size_t max_entries = 128) {
    if (ctx->graphs.size() <= max_entries) return;
    cudaDeviceSynchronize();
    for (auto& kv : ctx->graphs)
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    ctx->graphs.clear();
}
inline void graph_launch(acp_context* ctx, const std::string& key, cudaGraphExec_t e) {
    ACP_CUDA(cudaGraphLaunch(e, ctx->stream));
    ctx->launches += ctx->graphs[key].launches;
}

// ---- fft.cu -------------------------------------------------------------
FftPlan make_plan(int N);
void fft_init(acp_context* ctx);
void fft_free(acp_context* ctx);

// Which Fourier multiplier a Fourier-operator launch uses.
enum MultKind { MULT_KINETIC = 0, MULT_YUKAWA = 1, MULT_PRECOND = 2, MULT_NONE = 3 };

struct FopArgs {
    const double* X = nullptr;     // input columns (ld = Ng)
    double* Y = nullptr;           // output columns (ld = Ng); may alias X only if dots unused
    int n = 0;                     // number of columns
    const double* mult = nullptr;  // real multiplier per bin (already scaled by 1/N), or null
    const double* diag = nullptr;  // pointwise potential (Ng) or null
    const double* shift = nullptr; // per-column shift or null
    const int* active = nullptr;   // per-column activity flags or null
    double* dots = nullptr;        // per column: [0] x.y [1] x.x  (stride 2) or null
    long long* tprof = nullptr;    // debug: clock64() at phase boundaries of CTA 0 / thread 0, or null
    // Analytic symbol computed in-kernel from the bin index instead of a table read (saves the
    // per-CTA table traffic): -1 = use `mult`, MULT_KINETIC = |k|^2/2, MULT_PRECOND =
    // 1/(|k|^2/2 + tau) (preconditioner: reciprocal by rcp.approx + 2 Newton steps).
    int sym = -1;
    double tau = 0.0;
};
// Y = IFFT(mult * FFT(X)) + (diag - shift_j) (.) X, two real columns per complex FFT.
void fourier_op(acp_context* ctx, const FopArgs& a);
// Pre-allocate fourier_op's workspace for n columns (call before capturing it into a graph);
// alt = g: the workspace used while ctx->f2_alt == g (PCG node group g on its own stream).
void fourier_reserve(acp_context* ctx, int n, int alt);
// Fused 2D operator (fft2c.cu): square grids n = 16 N2, N2 in {2, 4, 8, 12, 16}.
bool f2c_supported(int n0, int n1);
size_t f2c_scratch_bytes(acp_context* ctx, int n);
size_t f2c_queue_ints(int n);
int f2c_items_per_phase(int N);
void launch_f2c(acp_context* ctx, const FopArgs& a, double2* S, int* queue, double* part, const double2* tw);
// Fill ctx->d_mult with a multiplier of the given kind (scaled by 1/N); returns it.
const double* multiplier(acp_context* ctx, MultKind kind, double tau);
// Real grid functions from Hermitian spectra given as complex coefficients per bin:
// out_j = (Ng/Omega) IFFT(spec_j)  (spec: Ng x n complex, bin-major per column).
void ifft_hermitian(acp_context* ctx, const double2* spec, int n, double* out);
// Spectrum out(k) = sum_a x(a) e^{-i k r_a} of one real column (bins in C order).
void real_spectrum(acp_context* ctx, const double* x, double2* out);
// Spectra of g_{I,a} (n = d*N_A columns, j = I*d + a) at positions R (device, N_A x d row-major).
void spectrum_G(acp_context* ctx, const double* d_R, double2* spec);
// Spectrum of the total pseudocharge m.
void spectrum_m(acp_context* ctx, const double* d_R, double2* spec);

// ---- gemm.cu ------------------------------------------------------------
// C (m x n, ld m) = alpha A^T B, A: K x m (lda), B: K x n (ldb); split-K partials reduced in order.
void gemm_tn(acp_context* ctx, int K, int m, int n, double alpha, const double* A, int lda,
             const double* B, int ldb, double* C);
// Partials only: Cp[z] (m x n) for the z-th K chunk of `kchunk` rows; returns the split count.
// The split pattern depends only on (K, kchunk), so per-column results do not depend on n.
int gemm_tn_partial(acp_context* ctx, int K, int m, int n, const double* A, int lda,
                    const double* B, int ldb, double* Cp, int kchunk);
int gemm_tn_splits(int K, int m, int n);
// C = beta C + alpha A B,  A: M x K (lda), B: K x n (ldb), C: M x n (ldc).
void gemm_nn(acp_context* ctx, int M, int K, int n, double alpha, const double* A, int lda,
             const double* B, int ldb, double beta, double* C, int ldc);

// ---- pcg.cu -------------------------------------------------------------
struct PcgStats {
    int max_iter = 0;
    long long total_iter = 0;
    double max_rel_res = 0.0;
    int n_solved = 0;
};
// Batched projected Sternheimer solve for columns j = c*nmu_p + mu:
// Q(H - shift_c)Q x = Q rhs_mu (rhs already in range(Q)).
void sternheimer_batch(acp_context* ctx, const double* Psi, int n_occ, const double* V,
                       const double* d_shift_c, int n_c, const double* rhs, int nmu_p,
                       double tol, int max_iter, double tau, double* X, PcgStats* st);
void apply_chi0(acp_context* ctx, const double* Psi, const double* eps, const double* V,
                const int* S, const double* Xi, int n_mu, int mu_begin, int mu_end, int n_cheb,
                double tol, int max_iter, double* W, PcgStats* st);

void kernel_bench(acp_context* ctx, int which, const double* Psi, const double* V, const double* X, int n,
                  double* Y, int reps);

// ---- qrcp.cu ------------------------------------------------------------
int compress(acp_context* ctx, const double* Psi, const double* Gp, int n_cols,
             const double* h_theta, const int* h_nu, int r_half, double id_eps, int n_fixed,
             int n_mu_max, int* S, double* Xi);

// ---- dense.cu -----------------------------------------------------------
// Solve A X = B in place (A: n x n col-major, B: n x nrhs col-major), partial pivoting.
void lu_solve(acp_context* ctx, double* A, int n, double* B, int nrhs);
// structured (Kronecker) QRCP for large sketches (qrcp_kron.cu)
bool kq_supported(int r);
int kq_compress(acp_context* ctx, const double* Psi, const double* Gt, int r, int kmax, double id_eps, int n_fixed,
                int n_mu_max, int* S, double* Xi);
// sharded QRCP (one pivot step per launch; the host all-gathers the candidates between steps)
int qrs_begin(acp_context* ctx, const double* Psi, const double* Gp, int n_cols, const double* h_theta,
              const int* h_nu, int r_half, int col_begin, int col_end, int n_fixed, int n_mu_max);
void qrs_step(acp_context* ctx, int s, const double* recv, int world, double id_eps, double* send);
void qrs_status(acp_context* ctx, int* stop, int* N);
int qrs_finish(acp_context* ctx, int* S, double* XiT);
// Same for [A | B] stored as ONE n x (n + nrhs) column-major array (multi-kernel blocked LU, any n).
void lu_solve_blocked(acp_context* ctx, double* AB, int n, int nrhs);
// U X = B for upper-triangular U stored as the first n columns of AB (n x (n + nrhs), ld n).
void upper_solve_blocked(acp_context* ctx, double* AB, int n, int nrhs);
// Symmetric eigenvalues (and optionally vectors) of A (n x n col-major, destroyed) by Jacobi.
void sym_eig(acp_context* ctx, double* A, int n, double* w, double* V);
// Cholesky A = L L^T in place (lower), returns false if not SPD.
void cholesky(acp_context* ctx, double* A, int n);

// ---- dyson / phonon / scf ----------------------------------------------
void smw_update(acp_context* ctx, const double* G, const int* S, const double* W, int N, double* U, double* Gp);
void dyson(acp_context* ctx, const double* Psi, const double* eps, const double* V, const double* G,
           const acp_dyson_opts& o, const double* h_theta, const int* h_nu, double* U, double* h_info);
void dynamical_matrix(acp_context* ctx, const double* h_R, const double* rho, const double* G,
                      const double* U, const double* h_masses, double* h_D, double* h_lambda);
void ground_state(acp_context* ctx, const double* h_R, const acp_scf_opts& o, double* Psi,
                  double* eps, double* rho, double* V, double* G, double* h_info);
void perturbations(acp_context* ctx, const double* h_R, double* G);

// ---- small device helpers ----------------------------------------------
void fill(acp_context* ctx, double* p, size_t n, double v);
void copy_cols(acp_context* ctx, double* dst, const double* src, size_t n);

}  // namespace acp
