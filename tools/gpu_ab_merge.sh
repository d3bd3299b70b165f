cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CONFIGS="c4;c5 --batch 256 --decode 128;c5 --batch 64 --decode 512" bash tools/gpu_perf.sh
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2b.log 2>&1; grep '"metric"' gpurun_out/bench_c2b.log | python tools/bench_brief.py
timeout 2400 python -m pytest tests -m gpu -q -rf -x > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/ab_pytest.log
