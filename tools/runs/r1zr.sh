mkdir -p gpurun_out
T=r1zr
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
ACP_PCG_HOSTLOOP=1 timeout 600 python bench.py --steps 1 --warmup 1 --skip-cpu > gpurun_out/${T}_plain.log 2>&1; echo "plain rc $?"
ACP_PCG_HOSTLOOP=1 timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_lu_panel_warp|k_proj_update" -s 40 -c 4 -o gpurun_out/${T}_full \
    python bench.py --steps 1 --warmup 1 --skip-cpu > gpurun_out/${T}_ncu.log 2>&1
echo "ncu rc $?"
