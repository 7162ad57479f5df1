# Heavy complex-payload timing (tools/heavy_ab.py) for each library variant
# present in the package directory (libotfx_*.so built with -D knobs); logs in
# gpurun_out/heavy_<variant>.log
for lib in paper_1712_10279_b200/libotfx*.so; do
  v=$(basename $lib .so)
  OTFX_LIB=$PWD/$lib timeout 400 python tools/heavy_ab.py > gpurun_out/heavy_$v.log 2>&1
  echo "== $v"; cat gpurun_out/heavy_$v.log
done
