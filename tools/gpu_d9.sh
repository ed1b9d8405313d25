mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_batch_gpu.py tests/test_fuzz.py tests/test_gpu_parity.py tests/test_multirank_gpu.py -x -q -p no:cacheprovider > gpurun_out/pytest_d9.log 2>&1; tail -3 gpurun_out/pytest_d9.log
bash tools/gpu_ncu_batch.sh d9 0x0
