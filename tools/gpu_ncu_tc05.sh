cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc05 -s 40 -c 1 -o gpurun_out/ncu_tc05b -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_tc05b.log 2>&1; echo rc $?
