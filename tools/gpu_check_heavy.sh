# GPU suite + heavy timing + bench (logs in gpurun_out/)
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 400 python tools/heavy_ab.py > gpurun_out/heavy.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
tail -3 gpurun_out/gputest.log; cat gpurun_out/heavy.log; tail -c 3000 gpurun_out/bench.log
