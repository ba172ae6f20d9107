mkdir -p gpurun_out
T=${TAG:-R2r}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_golden.py -q -x -k "full_m or kronecker or c2_1d" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/${T}_pytest.log
for C in c3g_2d_8x8 c4g_2d_16x16; do
for E in X=1; do
env ACP_KQ_PROF=1 ${E%%=*}=${E#*=} timeout 300 python tools/qr_time.py $C 1 > gpurun_out/${T}_q.log 2>&1; echo "$C $E $(grep -o '"ms": [0-9.]*' gpurun_out/${T}_q.log) $(grep kq gpurun_out/${T}_q.log | tail -1)"
done; done
