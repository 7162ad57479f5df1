# real-Lindblad commutator path A/B (OTFX_REAL_L=0/1) + matrix GPU tests
OTFX_REAL_L=0 timeout 400 python tools/heavy_ab.py > gpurun_out/heavy_rl0.log 2>&1
timeout 400 python tools/heavy_ab.py > gpurun_out/heavy_rl1.log 2>&1
OTFX_REAL_L=0 timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_rl0.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_rl1.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputest_rl.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_rl.log
echo rl0; cat gpurun_out/heavy_rl0.log; echo rl1; cat gpurun_out/heavy_rl1.log
for v in 0 1; do grep -o '"matrix_roofline": \[.*\]' gpurun_out/bench_rl$v.log | grep -o '"config": "[^"]*"\|"ms_per_iteration": [0-9.]*\|"frac": [0-9.]*' | paste - - - ; done
tail -3 gpurun_out/gputest_rl.log
