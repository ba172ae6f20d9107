# Round 2, call R3a: Kronecker QRCP without the Q^T a_c pass (coefficients from the R rows), 32 psi
# fragments in flight in the R-row pass; X placement by N_occ.  Full GPU suite, K3 timings, c4g bench
# with the QRCP phase profile.
mkdir -p gpurun_out
T=${TAG:-R3a}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/${T}_pytest.log
for w in 2 3; do timeout 300 python tools/k1_time.py c4g_2d_16x16 4096 10 $w 2>&1 | tail -1 | cut -c1-120; done
ACP_KQ_PROF=1 timeout 900 python bench.py --steps 3 --warmup 3 --skip-cpu > gpurun_out/${T}_bench.log 2>gpurun_out/${T}_bench.err; echo "bench rc $?"
grep '^{' gpurun_out/${T}_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['step_ms_each'], {k: round(v['us'],1) for k,v in d['kernels'].items()}, d['roofline']['kernel'], d['roofline']['frac'], d['e2e']['ms_each'], d['clocks'])"
grep -i "kq" gpurun_out/${T}_bench.err | sort | uniq -c | head -4
