"""Thin ctypes binding of include/acp_b200.h (argument marshalling only).

Every numerical step runs inside libacp_b200.so (hand-written sm_100a kernels).
There is no CPU fallback: importing this module raises if the library is
missing, and every call raises ``AcpError`` on a non-zero status.

Layout convention: a column-major N_g x n batch of grid functions (the C ABI's
layout) is a contiguous torch.float64 CUDA tensor of shape (n, N_g) -- row j of
the tensor is column j of the batch.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libacp_b200.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run `python -m paper_1605_08021_b200.build` "
                      "(there is no CPU fallback)")
_lib = ctypes.CDLL(LIB_PATH)

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)


class AcpError(RuntimeError):
    pass


class acp_system(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int), ("grid", ctypes.c_int * 2), ("cell", ctypes.c_double * 2),
                ("n_atoms", ctypes.c_int), ("n_occ", ctypes.c_int), ("occ", ctypes.c_double),
                ("Z", ctypes.c_double), ("sigma", ctypes.c_double), ("kappa", ctypes.c_double),
                ("eps0", ctypes.c_double)]


class acp_scf_opts(ctypes.Structure):
    _fields_ = [("scf_tol", ctypes.c_double), ("max_scf_iter", ctypes.c_int), ("n_extra", ctypes.c_int),
                ("history", ctypes.c_int), ("beta", ctypes.c_double), ("kerker_k0", ctypes.c_double),
                ("eig_tol", ctypes.c_double)]


class acp_dyson_opts(ctypes.Structure):
    _fields_ = [("n_cheb", ctypes.c_int), ("n_outer", ctypes.c_int), ("r_half", ctypes.c_int),
                ("id_eps", ctypes.c_double), ("n_mu_fixed", ctypes.c_int), ("cg_tol", ctypes.c_double),
                ("max_cg_iter", ctypes.c_int)]


_V = ctypes.c_void_p
_sig = {
    "acp_create": [ctypes.POINTER(acp_system), ctypes.c_int, ctypes.POINTER(_V)],
    "acp_destroy": [_V],
    "acp_last_error": [_V],
    "acp_set_stream": [_V, _V],
    "acp_version": [],
    "acp_kernel_launches": [_V],
    "acp_ground_state": [_V, _dp, ctypes.POINTER(acp_scf_opts), _V, _V, _V, _V, _V, _dp],
    "acp_perturbations": [_V, _dp, _V],
    "acp_compress": [_V, _V, _V, ctypes.c_int, _dp, _ip, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                     ctypes.c_int, _V, _V, _ip],
    "acp_qrs_begin": [_V, _V, _V, ctypes.c_int, _dp, _ip, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                      ctypes.c_int, _ip],
    "acp_qrs_step": [_V, ctypes.c_int, _V, ctypes.c_int, ctypes.c_double, _V],
    "acp_qrs_status": [_V, _ip, _ip],
    "acp_qrs_finish": [_V, _V, _V, _ip],
    "acp_apply_chi0": [_V, _V, _V, _V, _V, _V, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                       ctypes.c_double, ctypes.c_int, _V, _dp],
    "acp_dyson": [_V, _V, _V, _V, _V, ctypes.POINTER(acp_dyson_opts), _dp, _ip, _V, _dp],
    "acp_smw_update": [_V, _V, _V, _V, ctypes.c_int, _V, _V],
    "acp_dynamical_matrix": [_V, _dp, _V, _V, _V, _dp, _dp, _dp],
    "acp_fourier_apply": [_V, _V, ctypes.c_int, ctypes.c_int, ctypes.c_double, _V, _V, _V],
    "acp_gemm_tn": [_V, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double, _V, ctypes.c_int, _V,
                    ctypes.c_int, _V],
    "acp_sym_eigvals": [_V, ctypes.c_int, _V, _V],
    "acp_lu_solve": [_V, ctypes.c_int, ctypes.c_int, _V, _V],
    "acp_kernel_bench": [_V, ctypes.c_int, _V, _V, _V, ctypes.c_int, _V, ctypes.c_int],
    "acp_get_stream": [_V],
    "acp_gemm_nn": [_V, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double, _V, ctypes.c_int, _V,
                    ctypes.c_int, ctypes.c_double, _V, ctypes.c_int],
}
for _name, _args in _sig.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = ctypes.c_int
_lib.acp_last_error.restype = ctypes.c_char_p
_lib.acp_version.restype = ctypes.c_char_p
_lib.acp_kernel_launches.restype = ctypes.c_longlong
_lib.acp_get_stream.restype = ctypes.c_void_p

EXPORTED = list(_sig)


def version() -> str:
    return _lib.acp_version().decode()


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not (t.is_cuda and t.is_contiguous()):
        raise AcpError("expected a contiguous CUDA tensor")
    return ctypes.c_void_p(t.data_ptr())


def _chk(name: str, t, device: int, dtype=torch.float64, shape=None, min_numel=None):
    """Validate a device argument before its pointer crosses the C ABI: CUDA, contiguous, on the
    context's device, the expected dtype and shape (None entries = any extent)."""
    if t is None:
        return
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise AcpError(f"{name}: expected a CUDA tensor")
    if t.device.index != device:
        raise AcpError(f"{name}: tensor on cuda:{t.device.index}, context on cuda:{device}")
    if t.dtype != dtype:
        raise AcpError(f"{name}: expected {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise AcpError(f"{name}: expected a contiguous tensor")
    if shape is not None:
        if t.dim() != len(shape) or any(e is not None and e != d for e, d in zip(shape, t.shape)):
            raise AcpError(f"{name}: expected shape {tuple(shape)}, got {tuple(t.shape)}")
    if min_numel is not None and t.numel() < min_numel:
        raise AcpError(f"{name}: expected at least {min_numel} elements, got {t.numel()}")


def _i32(S: torch.Tensor) -> torch.Tensor:
    """Pivot indices as the int32 array the C ABI takes (the oracle hands out int64)."""
    return S.to(torch.int32).contiguous()


def _host(a, dtype=np.float64):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a, a.ctypes.data_as(_dp if dtype == np.float64 else _ip)


class Context:
    """One acp_context on one CUDA device (a system + its FFT plan and workspace)."""

    def __init__(self, dim: int, grid: Sequence[int], cell: Sequence[float], n_atoms: int, n_occ: int,
                 occ: float, Z: float, sigma: float, kappa: float, eps0: float, device: int = 0):
        if not torch.cuda.is_available():
            raise AcpError("CUDA device required (no CPU fallback)")
        g = list(grid) + [1] * (2 - len(grid))
        c = list(cell) + [0.0] * (2 - len(cell))
        self.sys = acp_system(dim, (ctypes.c_int * 2)(*g), (ctypes.c_double * 2)(*c), n_atoms, n_occ, occ, Z,
                              sigma, kappa, eps0)
        self.device = device
        self.Ng = int(np.prod(grid))
        self.n_occ = n_occ
        self.n_pert = dim * n_atoms
        self.dim = dim
        self._h = ctypes.c_void_p()
        torch.cuda.set_device(device)
        st = _lib.acp_create(ctypes.byref(self.sys), device, ctypes.byref(self._h))
        if st != 0:
            raise AcpError(f"acp_create failed with status {st}")

    @classmethod
    def from_config(cls, cfg, device: int = 0) -> "Context":
        return cls(cfg.dim, cfg.grid, cfg.cell, cfg.n_atoms, cfg.n_occ, cfg.occ, cfg.Z, cfg.sigma, cfg.kappa,
                   cfg.eps0, device)

    def close(self):
        if self._h:
            _lib.acp_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st: int, what: str):
        if st != 0:
            msg = _lib.acp_last_error(self._h).decode()
            raise AcpError(f"{what} failed (status {st}): {msg}")

    def _pre(self):
        torch.cuda.synchronize(self.device)

    def _empty(self, *shape, dtype=torch.float64):
        return torch.empty(*shape, dtype=dtype, device=f"cuda:{self.device}")

    @property
    def kernel_launches(self) -> int:
        return int(_lib.acp_kernel_launches(self._h))

    # -- 1. ground state -------------------------------------------------
    def ground_state(self, R, scf_tol=1e-12, max_scf_iter=400, n_extra=4, history=12, beta=0.5,
                     kerker_k0=0.5, eig_tol=1e-13, with_G=True):
        self._pre()
        Rh, Rp = _host(R)
        nb = self.n_occ + max(1, n_extra)
        Psi = self._empty(self.n_occ, self.Ng)
        eps = self._empty(nb)
        rho = self._empty(self.Ng)
        V = self._empty(self.Ng)
        G = self._empty(self.n_pert, self.Ng) if with_G else None
        info = np.zeros(4)
        o = acp_scf_opts(scf_tol, max_scf_iter, n_extra, history, beta, kerker_k0, eig_tol)
        self._check(_lib.acp_ground_state(self._h, Rp, ctypes.byref(o), _ptr(Psi), _ptr(eps), _ptr(rho), _ptr(V),
                                          _ptr(G), info.ctypes.data_as(_dp)), "acp_ground_state")
        return dict(Psi=Psi, eps=eps, rho=rho, V=V, G=G, n_iter=int(info[0]), residual=float(info[1]),
                    gap=float(info[2]))

    def perturbations(self, R) -> torch.Tensor:
        self._pre()
        Rh, Rp = _host(R)
        G = self._empty(self.n_pert, self.Ng)
        self._check(_lib.acp_perturbations(self._h, Rp, _ptr(G)), "acp_perturbations")
        return G

    # -- 2. compression --------------------------------------------------
    def compress(self, Psi, Gp, theta, nu, id_eps=1e-3, n_mu_fixed=0, n_mu_max=None):
        self._pre()
        _chk("Psi", Psi, self.device, shape=(self.n_occ, self.Ng))
        _chk("Gp", Gp, self.device, shape=(None, self.Ng))
        n_cols = Gp.shape[0]
        th, thp = _host(theta)
        nuh, nup = _host(nu, np.int32)
        if th.size != n_cols:
            raise AcpError(f"theta: expected {n_cols} draws, got {th.size}")
        r_half = len(nuh)
        if n_mu_max is None:
            n_mu_max = min(self.n_occ * 2 * r_half, self.Ng)
        S = self._empty(n_mu_max, dtype=torch.int32)
        Xi = self._empty(n_mu_max, self.Ng)
        nm = ctypes.c_int(0)
        self._check(_lib.acp_compress(self._h, _ptr(Psi), _ptr(Gp), n_cols, thp, nup, r_half, id_eps, n_mu_fixed,
                                      n_mu_max, _ptr(S), _ptr(Xi), ctypes.byref(nm)), "acp_compress")
        n = nm.value
        return S[:n].clone(), Xi[:n].clone(), n

    # -- 2'. sharded compression (multi-GPU driver: parallel.compress_sharded) ----
    def qrs_begin(self, Psi, Gp, theta, nu, col_begin, col_end, n_mu_fixed=0, n_mu_max=None):
        self._pre()
        _chk("Psi", Psi, self.device, shape=(self.n_occ, self.Ng))
        _chk("Gp", Gp, self.device, shape=(None, self.Ng))
        n_cols = Gp.shape[0]
        th, thp = _host(theta)
        nuh, nup = _host(nu, np.int32)
        if th.size != n_cols:
            raise AcpError(f"theta: expected {n_cols} draws, got {th.size}")
        if n_mu_max is None:
            n_mu_max = min(self.n_occ * 2 * len(nuh), self.Ng)
        m = ctypes.c_int(0)
        self._check(_lib.acp_qrs_begin(self._h, _ptr(Psi), _ptr(Gp), n_cols, thp, nup, len(nuh), col_begin, col_end,
                                       n_mu_fixed, n_mu_max, ctypes.byref(m)), "acp_qrs_begin")
        self._qrs = (col_begin, col_end, n_mu_max)
        return m.value

    def qrs_step(self, s: int, recv, world: int, id_eps: float, send):
        _chk("recv", recv, self.device)
        _chk("send", send, self.device)
        self._check(_lib.acp_qrs_step(self._h, s, _ptr(recv), world, id_eps, _ptr(send)), "acp_qrs_step")

    def qrs_status(self):
        st, n = ctypes.c_int(0), ctypes.c_int(0)
        self._check(_lib.acp_qrs_status(self._h, ctypes.byref(st), ctypes.byref(n)), "acp_qrs_status")
        return bool(st.value), n.value

    def qrs_finish(self):
        """-> (S (N_mu,) int32, XiT (col_end - col_begin, N_mu): this rank's rows of Xi, N_mu)."""
        b, e, n_mu_max = self._qrs
        S = self._empty(n_mu_max, dtype=torch.int32)
        XiT = self._empty(max(e - b, 1) * n_mu_max)
        n = ctypes.c_int(0)
        self._check(_lib.acp_qrs_finish(self._h, _ptr(S), _ptr(XiT), ctypes.byref(n)), "acp_qrs_finish")
        N = n.value
        return S[:N].clone(), XiT[: (e - b) * N].view(e - b, N), N

    # -- 3. compressed chi0 ----------------------------------------------
    def apply_chi0(self, Psi, eps, V, S, Xi, n_cheb, cg_tol=1e-11, max_iter=2000, mu_range=None, W=None):
        self._pre()
        n_mu = Xi.shape[0]
        S = _i32(S)
        mb, me = (0, n_mu) if mu_range is None else mu_range
        if W is None:
            W = torch.zeros(n_mu, self.Ng, dtype=torch.float64, device=Psi.device)
        _chk("Psi", Psi, self.device, shape=(self.n_occ, self.Ng))
        _chk("eps", eps, self.device, min_numel=self.n_occ)
        _chk("V", V, self.device, shape=(self.Ng,))
        _chk("S", S, self.device, dtype=torch.int32, shape=(n_mu,))
        _chk("Xi", Xi, self.device, shape=(n_mu, self.Ng))
        _chk("W", W, self.device, shape=(n_mu, self.Ng))
        info = np.zeros(4)
        eps_occ = eps[: self.n_occ].contiguous()
        self._check(_lib.acp_apply_chi0(self._h, _ptr(Psi), _ptr(eps_occ), _ptr(V), _ptr(S),
                                        _ptr(Xi), n_mu, mb, me, n_cheb, cg_tol, max_iter, _ptr(W),
                                        info.ctypes.data_as(_dp)), "acp_apply_chi0")
        return W, dict(max_iter=int(info[0]), total_iter=int(info[1]), max_rel_res=float(info[2]),
                       n_solved=int(info[3]))

    # -- 4. Dyson / Alg. 4 ----------------------------------------------
    def dyson(self, Psi, eps, V, G, n_cheb, n_outer, theta, nu, id_eps=1e-3, n_mu_fixed=0, cg_tol=1e-11,
              max_cg_iter=2000, U=None):
        self._pre()
        theta = np.ascontiguousarray(theta, dtype=np.float64)
        if theta.size != n_outer * self.n_pert:
            raise AcpError(f"theta: expected n_outer x dN_A = {n_outer * self.n_pert} draws, got {theta.size}")
        theta = theta.reshape(n_outer, -1)
        nu = np.ascontiguousarray(nu, dtype=np.int32)
        if nu.size % n_outer:
            raise AcpError(f"nu: {nu.size} frequencies do not split into {n_outer} outer iterations")
        nu = nu.reshape(n_outer, -1)
        _chk("Psi", Psi, self.device, shape=(self.n_occ, self.Ng))
        _chk("eps", eps, self.device, min_numel=self.n_occ)
        _chk("V", V, self.device, shape=(self.Ng,))
        _chk("G", G, self.device, shape=(self.n_pert, self.Ng))
        _chk("U", U, self.device, shape=(self.n_pert, self.Ng))
        r_half = nu.shape[1]
        o = acp_dyson_opts(n_cheb, n_outer, r_half, id_eps, n_mu_fixed, cg_tol, max_cg_iter)
        if U is None:
            U = self._empty(self.n_pert, self.Ng)
        info = np.zeros(8 + 3 * n_outer)
        eps_occ = eps[: self.n_occ].contiguous()
        self._check(_lib.acp_dyson(self._h, _ptr(Psi), _ptr(eps_occ), _ptr(V), _ptr(G), ctypes.byref(o),
                                   theta.ctypes.data_as(_dp), nu.ctypes.data_as(_ip), _ptr(U),
                                   info.ctypes.data_as(_dp)), "acp_dyson")
        per = info[8:].reshape(n_outer, 3)
        return U, dict(total_solves=int(info[0]), total_cg_iter=int(info[1]), max_cg_iter=int(info[2]),
                       max_rel_res=float(info[3]), n_mu=[int(x) for x in per[:, 0]],
                       diff=[float(x) for x in per[:, 1]], cg_iter=[int(x) for x in per[:, 2]])

    def smw_update(self, G, S, W, U=None, Gp=None):
        """Eq. dyson4: returns (U, Gp) with U = W Y, Gp = G + (K W) Y."""
        self._pre()
        S = _i32(S)
        _chk("G", G, self.device, shape=(self.n_pert, self.Ng))
        _chk("W", W, self.device, shape=(None, self.Ng))
        _chk("S", S, self.device, dtype=torch.int32, shape=(W.shape[0],))
        _chk("U", U, self.device, shape=(self.n_pert, self.Ng))
        _chk("Gp", Gp, self.device, shape=(self.n_pert, self.Ng))
        if U is None:
            U = self._empty(self.n_pert, self.Ng)
        if Gp is None:
            Gp = self._empty(self.n_pert, self.Ng)
        self._check(_lib.acp_smw_update(self._h, _ptr(G), _ptr(S), _ptr(W), W.shape[0], _ptr(U),
                                        _ptr(Gp)), "acp_smw_update")
        return U, Gp

    # -- 5. dynamical matrix --------------------------------------------
    def dynamical_matrix(self, R, rho, G, U, masses=None):
        self._pre()
        _chk("rho", rho, self.device, shape=(self.Ng,))
        _chk("G", G, self.device, shape=(self.n_pert, self.Ng))
        _chk("U", U, self.device, shape=(self.n_pert, self.Ng))
        if np.asarray(R).size != self.n_pert:
            raise AcpError(f"R: expected N_A x d = {self.n_pert} coordinates")
        Rh, Rp = _host(R)
        n = self.n_pert
        D = np.zeros((n, n))
        lam = np.zeros(n)
        mp = None
        if masses is not None:
            mh, mp = _host(masses)
        self._check(_lib.acp_dynamical_matrix(self._h, Rp, _ptr(rho), _ptr(G), _ptr(U), mp,
                                              D.ctypes.data_as(_dp), lam.ctypes.data_as(_dp)),
                    "acp_dynamical_matrix")
        return D.T.copy(), lam  # column-major -> row-major (D is symmetric anyway)

    # -- streams / timing -------------------------------------------------
    def stream_handle(self) -> int:
        """The raw cudaStream_t the library launches on (to restore after a temporary switch)."""
        return int(_lib.acp_get_stream(self._h) or 0)

    def set_stream_handle(self, handle: int):
        self._check(_lib.acp_set_stream(self._h, ctypes.c_void_p(handle) if handle else None), "acp_set_stream")

    def set_stream(self, stream: Optional["torch.cuda.Stream"]):
        """Launch on `stream` (a non-default torch stream, so graphs can be captured)."""
        self._check(_lib.acp_set_stream(self._h, None if stream is None else ctypes.c_void_p(stream.cuda_stream)),
                    "acp_set_stream")

    def kernel_bench(self, which: int, Psi, V, X, Y, reps: int):
        """Enqueue `reps` launches of hot kernel `which` (0: K1, 1: K2, 2: K3); no sync."""
        self._check(_lib.acp_kernel_bench(self._h, which, _ptr(Psi), _ptr(V), _ptr(X), X.shape[0], _ptr(Y), reps),
                    "acp_kernel_bench")

    # -- building blocks ------------------------------------------------
    def fourier_apply(self, X, which: int, tau: float = 0.0, diag=None, shift=None):
        self._pre()
        _chk("X", X, self.device, shape=(None, self.Ng))
        _chk("diag", diag, self.device, shape=(self.Ng,))
        _chk("shift", shift, self.device, shape=(X.shape[0],))
        Y = torch.empty_like(X)
        self._check(_lib.acp_fourier_apply(self._h, _ptr(X), X.shape[0], which, tau, _ptr(diag), _ptr(shift),
                                           _ptr(Y)), "acp_fourier_apply")
        return Y

    def gemm_tn(self, A, B, alpha=1.0):
        """C = alpha A^T B with A (K x m) and B (K x n) column-major -> returns tensor (n, m)."""
        self._pre()
        m, K = A.shape
        n = B.shape[0]
        C = self._empty(n, m)
        self._check(_lib.acp_gemm_tn(self._h, K, m, n, alpha, _ptr(A), K, _ptr(B), K, _ptr(C)), "acp_gemm_tn")
        return C

    def lu_solve(self, A, B):
        """X with A X = B for column-major A (n x n: tensor (n, n) holding A^T) and B (n x nrhs:
        tensor (nrhs, n)); returns (LU factors, X) as new tensors in the same layout."""
        self._pre()
        A = A.clone()
        B = B.clone()
        n = A.shape[0]
        nrhs = B.shape[0]
        self._check(_lib.acp_lu_solve(self._h, n, nrhs, _ptr(A), _ptr(B)), "acp_lu_solve")
        return A, B

    def sym_eigvals(self, A):
        """Ascending eigenvalues of the symmetric matrix A (n x n tensor on the device)."""
        self._pre()
        n = A.shape[0]
        w = self._empty(n)
        self._check(_lib.acp_sym_eigvals(self._h, n, _ptr(A), _ptr(w)), "acp_sym_eigvals")
        return w

    def gemm_nn(self, A, B, C=None, alpha=1.0, beta=0.0):
        """C = beta C + alpha A B, A (M x K) column-major = tensor (K, M); B (K x n) = tensor (n, K)."""
        self._pre()
        K, M = A.shape
        n = B.shape[0]
        if C is None:
            C = torch.zeros(n, M, dtype=torch.float64, device=A.device)
        self._check(_lib.acp_gemm_nn(self._h, M, K, n, alpha, _ptr(A), M, _ptr(B), K, beta, _ptr(C), M),
                    "acp_gemm_nn")
        return C
