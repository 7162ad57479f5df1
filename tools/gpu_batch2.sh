timeout 1200 python -m pytest tests/test_gpu_channel_counts.py -q -x > gpurun_out/channel_counts.log 2>&1; echo "channel rc=$?" >> gpurun_out/channel_counts.log
bash tools/gpu_sanitize.sh
