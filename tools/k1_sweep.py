"""Time the K1 Fourier operator (H apply: kinetic symbol + potential, the PCG's H p launch)
for the bench shapes, sweeping the CTA size knob ACP_FFT_THREADS.  CUDA-event timing, warm.

  python tools/k1_sweep.py [config] [ncols] [T1,T2,...]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from workloads import get_config  # noqa: E402
from paper_1605_08021_b200 import Context  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c1_1d_insulator"
    ncols = int(sys.argv[2]) if len(sys.argv) > 2 else 928
    Ts = [int(t) for t in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0]
    cfg = get_config(name)
    for T in Ts:
        if T:
            os.environ["ACP_FFT_THREADS"] = str(T)
        else:
            os.environ.pop("ACP_FFT_THREADS", None)
        ctx = Context.from_config(cfg)
        s = torch.cuda.Stream()
        ctx.set_stream(s)
        Psi = torch.randn(cfg.n_occ, cfg.n_grid, dtype=torch.float64, device="cuda")
        V = torch.randn(cfg.n_grid, dtype=torch.float64, device="cuda")
        X = torch.randn(ncols, cfg.n_grid, dtype=torch.float64, device="cuda")
        Y = torch.zeros_like(X)
        ctx.kernel_bench(0, Psi, V, X, Y, 3)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record(s)
        ctx.kernel_bench(0, Psi, V, X, Y, reps)
        e1.record(s)
        torch.cuda.synchronize()
        us = 1e3 * e0.elapsed_time(e1) / reps
        gbs = 16.0 * cfg.n_grid * ncols / us / 1e3
        print(json.dumps({"config": name, "ncols": ncols, "T": T or "default", "us": us, "GBps": gbs}), flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
