# round-end evidence: smoke, bench (both arms), headline ncu (launch list +
# full capture), heavy-payload ncu; logs in gpurun_out/
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
timeout 1200 bash tools/profile.sh r02c > gpurun_out/profile.log 2>&1
python tools/matrix_probe.py c3k3 2048 260 > gpurun_out/heavy_probe_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep_tma -s 255 -c 1 \
    -o gpurun_out/r02c_heavy python tools/matrix_probe.py c3k3 2048 260 > gpurun_out/heavy_ncu.log 2>&1
tail -2 gpurun_out/smoke.log; tail -c 800 gpurun_out/bench.log; tail -c 600 gpurun_out/bench_ref.log; tail -2 gpurun_out/profile.log; tail -2 gpurun_out/heavy_ncu.log
