# small-grid timing (BASELINE C1-C4 sizes), GPU suite, and an ncu launch list +
# full capture of the 256^2 register sweep (host run loop: ncu cannot profile
# kernels inside conditional graphs); logs in gpurun_out/
SIZES=128,256,512 timeout 600 python tools/small_grid_timing.py '{}' > gpurun_out/small_vector.log 2>&1
timeout 600 python tools/matrix_small_timing.py '{}' > gpurun_out/small_matrix.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
export OTFX_DEVICE_LOOP=0
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/small_launches.csv python tools/small_probe.py > gpurun_out/small_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 150 -c 1 -o gpurun_out/small_sweep python tools/small_probe.py > gpurun_out/small_ncu_full.log 2>&1
cat gpurun_out/small_vector.log gpurun_out/small_matrix.log; tail -3 gpurun_out/gputest.log; tail -2 gpurun_out/small_ncu_full.log
