mkdir -p gpurun_out
python -m pytest tests/test_fuzz.py tests/test_gpu_parity.py tests/test_ctx_gpu.py -x -q -m gpu -p no:cacheprovider > gpurun_out/pytest8.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest8.log
tail -3 gpurun_out/pytest8.log
python tools/sweep_encode.py 3 0x0 0x80000 > gpurun_out/sweep8_enc3.log 2>&1
python tools/sweep_encode.py 2 0x0 0x100000 > gpurun_out/sweep8_enc2.log 2>&1
cat gpurun_out/sweep8_enc3.log gpurun_out/sweep8_enc2.log
