# A/B of programmatic dependent launch (OTFX_PDL=0/1): small-grid vector and
# matrix solves (BASELINE C1-C4 sizes) and the headline bench; logs in gpurun_out/
SIZES=128,256,512 timeout 600 python tools/small_grid_timing.py '{"OTFX_PDL":"0"}' '{"OTFX_PDL":"1"}' > gpurun_out/pdl_vector.log 2>&1
timeout 600 python tools/matrix_small_timing.py '{"OTFX_PDL":"0"}' '{"OTFX_PDL":"1"}' > gpurun_out/pdl_matrix.log 2>&1
cat gpurun_out/pdl_vector.log gpurun_out/pdl_matrix.log
