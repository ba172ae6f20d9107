"""bench.py -- time the ACP hot path (Alg. 4 + dynamical matrix) on B200.

One STEP = the whole hot path on one synthetic system: n_outer outer iterations of
Alg. 4 (compress with SRFT + QRCP, N_c x N_mu projected Sternheimer solves, W,
SMW update) followed by the dynamical-matrix assembly and its eigenvalues.  The
ground state is prepared once, untimed (it is the input of the hot path).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME] [--impl acp|reference]

Metric (BASELINE.json): Sternheimer solves/s (whole job), with time-to-D in ms
and the roofline fraction of the dominant kernel.  Multi-GPU runs (torchrun) shard
the mu-columns of every outer iteration across ranks and all-gather W over NCCL.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ACP dynamical-matrix time-to-solution; Sternheimer solves/s; % HBM roofline"
L2_BYTES = 126 * 1024 * 1024


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    d = json.load(open(p)) if os.path.exists(p) else {}
    hbm = d.get("hbm_gbs")
    bf16 = d.get("bf16_tflops")
    src = "measured (MEASURED_PEAKS.json)"
    if hbm is None:
        hbm, bf16, src = 6650.0, 1590.0, "fallback (B200_PROFILING.md)"
    # FP64 peak MEASURED on this pool's B200 (tools/micro/fp64_peak.cu, profiles/R2a_fp64_peak_b200.txt):
    # DMMA (mma.sync .f64, every shape) 37.1 TF/s, DFMA 36.4 TF/s -- the driver's file has no FP64 entry
    fp64 = 37.1
    return dict(hbm_gbs=hbm, fp64_tflops=fp64, src=src, fp64_src="measured (profiles/R2a_fp64_peak_b200.txt)")


class ClockSampler:
    """nvidia-smi sampling during the timed region (clocks + throttle reasons)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.f = tempfile.NamedTemporaryFile(mode="w+", suffix=".csv", delete=False)
        if os.environ.get("ACP_BENCH_NO_SMI"):  # diagnostics: no sampler process
            self.p = None
            return
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(device), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.15)
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [float(r[0]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(rows[0][1]), "samples": len(rows),
                "reasons": reasons}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------------ oracle (reference arm / cpu baseline)
DENSE_MAX_NG = 6000   # the dense oracle (N_g x N_g matrices) runs up to configs[2]


def oracle_sample(cfg, R, outer_k: int = 0, state=None):
    """A bounded sample of the oracle on this workload.

    N_g <= 6000: one outer iteration of the oracle's Alg. 4 (compress + direct compressed solves
    + W + SMW) on its own dense ground state.  2D grids: the oracle's MINRES solves of Eq.
    eqncompressU (oracle/iterative.py) for 16 interpolation vectors of outer iteration 0 at one
    Chebyshev node per sample, on the oracle's cached ground state (tests/cache, written by
    tools/make_golden.py).  Returns (seconds, solves, state, description)."""
    from workloads import sketch_draws
    from oracle.model import Model
    from oracle import acp as oacp
    if cfg.n_grid <= DENSE_MAX_NG:
        from oracle.scf import scf
        if state is None:
            m = Model(cfg, R)
            gs = scf(m, tol=max(cfg.scf_tol, 1e-10))   # untimed input; the dense SCF stalls near 1e-11 on configs[2]
            state = dict(m=m, gs=gs, H=m.hamiltonian_dense(gs.V), G=m.G_matrix())
        m, gs, H, G = state["m"], state["gs"], state["H"], state["G"]
        th, nu = sketch_draws(cfg.seed, outer_k % cfg.n_outer, G.shape[1], cfg.sketch_r)
        t0 = time.perf_counter()
        S, Xi, _ = oacp.compress(m, gs.Psi, G, th, nu, cfg.id_eps)
        W = oacp.compressed_W(m, H, gs.Psi, gs.eps[: cfg.n_occ], S, Xi, cfg.n_cheb)
        oacp.smw_update(m, G, W, S)
        dt = time.perf_counter() - t0
        return dt, cfg.n_cheb * len(S), state, (f"one outer iteration of the dense oracle's Alg. 4 "
                                                 f"(compress + {cfg.n_cheb} x N_mu direct solves + W + SMW)")
    from oracle.iterative import SternheimerMinres
    if state is None:
        gp = os.path.join(ROOT, "tests", "cache", f"{cfg.name}_gs.npz")
        xp = os.path.join(ROOT, "tests", "cache", f"{cfg.name}_xi0.npz")
        m = Model(cfg, R)
        if os.path.exists(gp) and os.path.exists(xp):
            z = np.load(gp)
            Psi, V, eo, Xi = z["Psi"], z["V"], z["eps"][: cfg.n_occ], np.load(xp)["Xi"][:, :16]
            src = "the oracle's ground state (tests/cache, tools/make_golden.py)"
        else:
            # without the cached oracle ground state (it is git-ignored: up to 134 MB): a stand-in
            # of the same shapes -- the N_occ lowest real plane waves (exact eigenvectors of H at
            # V = 0) and 16 seeded interpolation-vector-like columns; same operator sizes per solve
            sys.path.insert(0, os.path.join(ROOT, "tests"))
            from free_electron import plane_wave_ground_state
            m2 = 1
            while True:
                Psi, eps, _ = plane_wave_ground_state(cfg.grid, cfg.cell, m2)
                if Psi.shape[1] >= cfg.n_occ:
                    break
                m2 += 1
            Psi, eo, V = Psi[:, : cfg.n_occ], eps[: cfg.n_occ], np.zeros(m.Ng)
            Xi = np.random.default_rng(cfg.seed).standard_normal((m.Ng, 16))
            src = "a free-electron stand-in ground state of the same shapes (oracle cache absent)"
        state = dict(solver=SternheimerMinres(m, V, Psi, tol=cfg.cg_tol, block=16), Xi=Xi, src=src,
                     nodes=oacp.chebyshev_nodes(eo[0], eo[-1], cfg.n_cheb))
    c = outer_k % cfg.n_cheb
    t0 = time.perf_counter()
    state["solver"](state["nodes"][c], state["Xi"])
    dt = time.perf_counter() - t0
    return dt, state["Xi"].shape[1], state, ("the oracle's MINRES solves of Eq. eqncompressU (oracle/iterative.py, "
                                             "relative residual 1e-11) for 16 interpolation vectors of outer "
                                             "iteration 0 at one Chebyshev node per step, on " + state["src"])


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        n = [d.get("num_threads", 1) for d in threadpool_info() if d.get("user_api") == "blas"]
        return int(max(n)) if n else 1
    except Exception:
        return os.cpu_count() or 1


def run_reference(args, cfg):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from workloads import atom_positions
    R = atom_positions(cfg)
    state = None
    try:
        for _ in range(args.warmup):
            _, _, state, _ = oracle_sample(cfg, R, 0, state)
    except FileNotFoundError as e:
        print(json.dumps({"impl": "reference", "unavailable": str(e)}), flush=True)
        return
    tot_t, tot_s = 0.0, 0
    for k in range(args.steps):
        dt, ns, state, what = oracle_sample(cfg, R, k, state)
        tot_t += dt
        tot_s += ns
    v = tot_s / tot_t
    cores = blas_threads()
    sample = what + " (each step one such sample)"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "solves/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": cfg.name},
            "cpu_baseline": {"value": v, "unit": "solves/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
def run_acp(args, cfg):
    import torch
    import torch.distributed as dist
    from workloads import atom_positions, sketch_draws
    from paper_1605_08021_b200 import Context
    from paper_1605_08021_b200.parallel import dyson_sharded

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    sharded = world > 1 or args.dist
    if sharded:
        if world == 1 and "MASTER_ADDR" not in os.environ:
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(29500 + os.getpid() % 1000), RANK="0",
                              WORLD_SIZE="1")
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    dev = torch.device(f"cuda:{local}")
    ctx = Context.from_config(cfg, device=local)
    stream = torch.cuda.Stream(device=dev)
    ctx.set_stream(stream)
    R = atom_positions(cfg)
    t0 = time.perf_counter()
    gs = ctx.ground_state(R, scf_tol=cfg.scf_tol)
    t_gs = time.perf_counter() - t0
    n = cfg.n_pert
    dr = [sketch_draws(cfg.seed, k, n, cfg.sketch_r) for k in range(cfg.n_outer)]
    th = np.stack([d[0] for d in dr])
    nu = np.stack([d[1] for d in dr])
    Psi, eps, V, rho, G = gs["Psi"], gs["eps"], gs["V"], gs["rho"], gs["G"]
    flush = torch.empty(2 * L2_BYTES // 8, dtype=torch.float64, device=dev)

    def step():
        if sharded:
            with torch.cuda.stream(stream):  # torch ops, NCCL and the library on the timed stream
                U, info = dyson_sharded(ctx, Psi, eps, V, G, cfg.n_cheb, cfg.n_outer, lambda k: dr[k], cfg.id_eps,
                                    cfg.cg_tol, shard_compress={"auto": None, "on": True, "off": False}[args.shard_compress])
            solves = info["local_solves"]
            t = torch.tensor([solves], device=dev)
            dist.all_reduce(t)
            solves = int(t.item())
            info = dict(total_solves=solves, n_mu=info["n_mu"], compression=info["compression"])
        else:
            U, info = ctx.dyson(Psi, eps, V, G, cfg.n_cheb, cfg.n_outer, th, nu, id_eps=cfg.id_eps,
                                cg_tol=cfg.cg_tol)
        D, lam = ctx.dynamical_matrix(R, rho, G, U)
        return info, D, lam

    def barrier():
        if sharded:
            dist.barrier()
        torch.cuda.synchronize(dev)

    clocks = None
    for w in range(args.warmup):
        if w == args.warmup - 1:
            # the nvidia-smi sampler starts during the last warm-up step (its start-up is not in the
            # timed region); it samples until the timed steps end
            clocks = ClockSampler(local)
        step()
    if clocks is None:
        clocks = ClockSampler(local)
    # ---- timed region: device time per step (CUDA events on the launching stream), L2 flushed between steps
    launches0 = ctx.kernel_launches
    times = []
    solves = 0
    info = None
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.nvtx.range_push("acp_step")
        e0.record(stream)
        info, D, lam = step()
        e1.record(stream)
        torch.cuda.nvtx.range_pop()
        barrier()
        times.append(e0.elapsed_time(e1))
        solves += info["total_solves"]
    launches = ctx.kernel_launches - launches0
    clk = clocks.stop()
    t_ms = float(np.sum(times))
    if sharded:
        tt = torch.tensor([t_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
    value = solves / (t_ms / 1e3)

    # ---- e2e through the public API with HOST buffers (pinned), copies inside the timed region
    host = {k: v.cpu().pin_memory() for k, v in dict(Psi=Psi, eps=eps, V=V, rho=rho, G=G).items()}
    dev_in = {k: torch.empty_like(v, device=dev) for k, v in host.items()}
    h2d = int(sum(v.numel() * v.element_size() for v in host.values()))
    d2h = 8 * (n * n + n)
    e2e_ms = 0.0
    e2e_each = []
    e2e_steps = max(1, min(args.steps, 3))
    # one untimed pass first: the device input buffers are new allocations, so the PCG graphs
    # (keyed by their pointers) are captured here rather than inside the timed passes
    for it in range(e2e_steps + 1):
        with torch.cuda.stream(stream):
            flush.zero_()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        with torch.cuda.stream(stream):
            for k in host:
                dev_in[k].copy_(host[k], non_blocking=True)
        if sharded:
            with torch.cuda.stream(stream):
                U, inf2 = dyson_sharded(ctx, dev_in["Psi"], dev_in["eps"], dev_in["V"], dev_in["G"], cfg.n_cheb,
                                    cfg.n_outer, lambda k: dr[k], cfg.id_eps, cfg.cg_tol)
        else:
            U, inf2 = ctx.dyson(dev_in["Psi"], dev_in["eps"], dev_in["V"], dev_in["G"], cfg.n_cheb, cfg.n_outer,
                                th, nu, id_eps=cfg.id_eps, cg_tol=cfg.cg_tol)
        D2, lam2 = ctx.dynamical_matrix(R, dev_in["rho"], dev_in["G"], U)   # D, lambda land in host memory
        e1.record(stream)
        barrier()
        if it > 0:
            e2e_ms += e0.elapsed_time(e1)
            e2e_each.append(round(e0.elapsed_time(e1), 3))
    e2e_ms /= e2e_steps
    e2e_value = (solves / args.steps) / (e2e_ms / 1e3)

    # ---- live roofline of the hot kernels (same shapes as inside the step)
    peaks = _peaks()
    n_mu = info["n_mu"][0]
    # the production launch shape: one PCG node group's columns (pcg.cu: up to 4 groups on their own
    # streams when N_c N_mu' N_g <= 16M points, else one group = the whole batch)
    n_all = cfg.n_cheb * ((n_mu + 1) // 2 * 2)
    ngroups = min(cfg.n_cheb, 4) if n_all * ctx.Ng <= (16 << 20) else 1
    ncols = (cfg.n_cheb // ngroups) * ((n_mu + 1) // 2 * 2)
    nmu_p = (n_mu + 1) // 2 * 2
    sweep = int(os.environ.get("ACP_PCG_SWEEP", -1))
    if sweep < 0:  # pcg.cu's node sweep: large batches (N_mu' >= 768) run one Chebyshev node per warm-started group
        sweep = 1 if (ngroups == 1 and cfg.n_cheb >= 3 and nmu_p >= 768) else 0
    if 0 < sweep < cfg.n_cheb:
        ncols = sweep * nmu_p
    # X and Y for the kernel timing must fit beside the library's PCG workspace
    free_b, _ = torch.cuda.mem_get_info(dev)
    fit = int((free_b - (4 << 30)) // (2 * 8 * ctx.Ng)) // 2 * 2
    shape_note = "production launch shape (one PCG node group" + (f": {sweep} Chebyshev node(s) of the sweep)" if 0 < sweep < cfg.n_cheb else ")")
    if fit < ncols:
        ncols = max(2, fit)
        shape_note = (f"{ncols} of the production launch's {n_all} columns (memory beside the PCG workspace); "
                      f"per-column work and traffic are the same at any width >> SM count")
    X = torch.randn(ncols, ctx.Ng, dtype=torch.float64, device=dev)
    Y = torch.zeros_like(X)
    kern = {}
    reps = 50
    for which, name in [(0, "K1_fourier_op"), (1, "K2_gemm_tn"), (2, "K3_pcg_update")]:
        ctx.kernel_bench(which, Psi, V, X, Y, reps)  # warm-up; captures the reps-launch CUDA graph
        torch.cuda.synchronize(dev)
        with torch.cuda.stream(stream):
            flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ctx.kernel_bench(which, Psi, V, X, Y, reps)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        us = 1e3 * e0.elapsed_time(e1) / reps
        Ng, No = ctx.Ng, cfg.n_occ
        if which == 0:
            byts = 16.0 * Ng * ncols
            kern[name] = dict(bound="hbm", us=us, bytes=byts, achieved=byts / us / 1e3, unit="GB/s",
                              peak=peaks["hbm_gbs"])
            # the same launch seen as FP64 ALU work: two length-N_g FFTs per packed column pair,
            # 5 N log2 N flops each (complex radix-2 count), i.e. 5 N_g log2 N_g per real column
            fl = 5.0 * Ng * np.log2(Ng) * ncols
            kern[name]["alu"] = dict(flops=fl, achieved=fl / us / 1e6, unit="TFLOP/s", peak=peaks["fp64_tflops"],
                                     frac=fl / us / 1e6 / peaks["fp64_tflops"])
        elif which == 1:
            fl = 2.0 * Ng * No * ncols
            kern[name] = dict(bound="tensor", us=us, flops=fl, achieved=fl / us / 1e6, unit="TFLOP/s",
                              peak=peaks["fp64_tflops"])
        else:
            # Y - Psi C fused with the PCG axpys: 24 N_g bytes (EpBeta) and 2 N_g N_occ DMMA flops per
            # column.  Arithmetic intensity N_occ / 12 flop/B against the FP64 ridge (peak flops / HBM):
            # HBM-bound for N_occ = 32 (configs[1]), tensor-bound for N_occ >= 128 (configs[2], [4])
            byts = 24.0 * Ng * ncols
            fl = 2.0 * Ng * No * ncols
            hbm = dict(bound="hbm", us=us, bytes=byts, achieved=byts / us / 1e3, unit="GB/s", peak=peaks["hbm_gbs"])
            ten = dict(bound="tensor", us=us, flops=fl, achieved=fl / us / 1e6, unit="TFLOP/s",
                       peak=peaks["fp64_tflops"])
            ridge = peaks["fp64_tflops"] * 1e3 / peaks["hbm_gbs"]
            if fl / byts >= ridge:
                kern[name] = dict(ten, hbm=dict(hbm, frac=hbm["achieved"] / hbm["peak"]))
            else:
                kern[name] = dict(hbm, tensor=dict(ten, frac=ten["achieved"] / ten["peak"]))
        kern[name]["frac"] = kern[name]["achieved"] / kern[name]["peak"]
    # the dominant kernel = the largest share of the step: K1, K2 and K3 each launch twice per CG
    # iteration over the same columns (H p and M r; the two projections; EpAlpha and EpBeta), so
    # the share follows the per-launch time (K1 at configs[1], K3 at c4g)
    dom_name = os.environ.get("ACP_DOMINANT_KERNEL") or max(kern, key=lambda k: kern[k]["us"])
    dom = kern[dom_name]
    # DRAM bytes per launch of this kernel on THIS workload from one ncu --set full capture
    # (profiles/traffic.json: {workload: {kernel: {"bytes_per_launch", "units_per_launch", ...}}}),
    # scaled to this launch's width; null when no capture of this workload exists
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        ent = json.load(open(tf)).get(cfg.name, {}).get(dom_name)
        if ent:
            traffic = ent["bytes_per_launch"] * ncols / ent["units_per_launch"]
    roofline = {"kernel": dom_name, "bound": dom["bound"], "achieved": dom["achieved"], "peak": dom["peak"],
                "unit": dom["unit"], "frac": dom["frac"], "traffic": traffic, "peak_source": peaks["src"],
                "units_per_launch": ncols, "launch_shape": shape_note,
                "fp64_peak_source": peaks["fp64_src"], "per_unit": ("16*N_g bytes" if dom["bound"] == "hbm" and
                                                        dom_name.startswith("K1") else
                                                        "24*N_g bytes" if dom["bound"] == "hbm" else
                                                        "2*N_g*N_occ flops")}

    # ---- CPU baseline: the oracle, bounded sample (~10-30 s of host work), rank 0 at N = 1 only
    cpu = None
    if world == 1 and rank == 0 and not args.skip_cpu:
        try:
            st, tt, ns_tot, k = None, 0.0, 0, 0
            while tt < 10.0 and k < 64:
                dt, ns, st, what = oracle_sample(cfg, R, k, st)
                if k > 0 or cfg.n_grid <= DENSE_MAX_NG:  # first MINRES sample warms the FFT plans
                    tt += dt
                    ns_tot += ns
                k += 1
            cpu = {"value": ns_tot / tt, "unit": "solves/s", "cores": blas_threads(), "kind": "oracle",
                   "sample": f"{what}; {ns_tot} solves in {tt:.1f} s; ground state untimed"}
        except FileNotFoundError as e:
            cpu = {"value": None, "unit": "solves/s", "cores": blas_threads(), "kind": "oracle",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "time_to_D_ms": t_ms / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": cfg.name, "N_g": ctx.Ng, "N_A": cfg.n_atoms, "N_occ": cfg.n_occ,
                           "N_c": cfg.n_cheb, "n_outer": cfg.n_outer, "id_eps": cfg.id_eps, "r": cfg.sketch_r,
                           "cg_tol": cfg.cg_tol, "n_mu": info["n_mu"], "solves_per_step": solves // args.steps,
                           "l2": "flushed (256 MiB write) between timed steps",
                           "ground_state_s": round(t_gs, 2), "parallelism": (f"rhs shard x{world} (NCCL all-gather of W), compression {info.get('compression', '?')}" if sharded else "single GPU")},
                "roofline": roofline, "kernels": kern, "cpu_baseline": cpu,
                "step_ms_each": [round(t, 3) for t in times],
                "e2e": {"value": e2e_value, "unit": "solves/s", "ms_per_step": e2e_ms, "ms_each": e2e_each,
                        "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": d2h},
                "gpu_launches": int(launches), "clocks": clk}
        print(json.dumps(line), flush=True)
    if sharded:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    # default: the largest single-GPU configuration (BASELINE.json configs[4], 2D 16 x 16 on 256^2,
    # run with eps0 = 1: DESIGN.md reading R13); configs[1] is the secondary line (--config c1_1d_insulator)
    ap.add_argument("--config", default="c4g_2d_16x16")
    ap.add_argument("--impl", default="acp", choices=["acp", "reference"])
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--dist", action="store_true",
                    help="run the multi-GPU code path (sharded compression, NCCL all-gathers) even at N = 1")
    ap.add_argument("--shard-compress", default="auto", choices=["auto", "on", "off"],
                    help="multi-GPU path: Alg. 2 sharded by grid point (on), replicated (off), or the measured "
                         "rule of parallel.use_sharded_compress (auto: replicated up to 8 ranks)")
    args = ap.parse_args()
    from workloads import get_config
    cfg = get_config(args.config)
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_acp(args, cfg)


if __name__ == "__main__":
    main()
