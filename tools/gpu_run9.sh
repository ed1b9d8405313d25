mkdir -p gpurun_out
python -m pytest tests/test_batch_gpu.py tests/test_fuzz.py tests/test_batch_host.py -x -q -m gpu -p no:cacheprovider > gpurun_out/pytest9.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest9.log
tail -3 gpurun_out/pytest9.log
python tools/sweep_batch.py 4 1.0 0x0 > gpurun_out/sweep9_b4.log 2>&1
python tools/sweep_batch.py 5 1.0 0x0 > gpurun_out/sweep9_b5.log 2>&1
cat gpurun_out/sweep9_b4.log gpurun_out/sweep9_b5.log
