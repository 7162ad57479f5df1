timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-secondary > gpurun_out/bench_dual2.log 2>&1
OTFX_LIB=$PWD/paper_1712_10279_b200/libotfx_dual1.so timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-secondary > gpurun_out/bench_dual1.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
for v in 2 1; do tail -1 gpurun_out/bench_dual$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('minB', $v, d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['step_frac'])"; done
tail -3 gpurun_out/gputest.log
