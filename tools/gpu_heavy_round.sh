# GPU suite, heavy-payload timing (+ rows-per-CTA sweep), bench, and one ncu
# capture of the heavy complex sweep (3x3 complex l1nuc 2048^2); logs in gpurun_out/
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 400 python tools/heavy_ab.py > gpurun_out/heavy.log 2>&1
for R in 12 24 32; do OTFX_TILE_ROWS=$R timeout 400 python tools/heavy_ab.py > gpurun_out/heavy_rows$R.log 2>&1; done
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
python tools/matrix_probe.py c3k3 2048 260 > gpurun_out/heavy_probe_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep_tma -s 255 -c 1 \
    -o gpurun_out/r02_heavy_self8 python tools/matrix_probe.py c3k3 2048 260 > gpurun_out/heavy_ncu.log 2>&1
tail -3 gpurun_out/gputest.log; cat gpurun_out/heavy.log; for R in 12 24 32; do echo "rows $R"; cat gpurun_out/heavy_rows$R.log; done; tail -c 1500 gpurun_out/bench.log; tail -3 gpurun_out/heavy_ncu.log
