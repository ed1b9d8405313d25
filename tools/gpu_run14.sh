mkdir -p gpurun_out
python -m pytest tests/test_fuzz.py tests/test_batch_gpu.py -x -q -m gpu -p no:cacheprovider > gpurun_out/pytest14.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest14.log
tail -2 gpurun_out/pytest14.log
python tools/sweep_encode.py 3 0x0 > gpurun_out/sweep14.log 2>&1
python tools/sweep_encode.py 2 0x0 >> gpurun_out/sweep14.log 2>&1
python tools/sweep_batch.py 4 1.0 0x0 >> gpurun_out/sweep14.log 2>&1
python tools/sweep_batch.py 5 1.0 0x0 >> gpurun_out/sweep14.log 2>&1
cat gpurun_out/sweep14.log
