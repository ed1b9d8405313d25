mkdir -p gpurun_out
#python -m pytest tests/test_batch_gpu.py tests/test_fuzz.py tests/test_batch_host.py tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider -k "not full" > gpurun_out/pytest10.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest10.log
tail -3 gpurun_out/pytest10.log
python tools/sweep_batch.py 4 1.0 0x0 0x100 > gpurun_out/sweep10_b4.log 2>&1; python tools/sweep_batch.py 4 0.25 0x0 >> gpurun_out/sweep10_b4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"decode_batch3" -s 1 -c 1 -o gpurun_out/b3_lm python tools/sweep_batch.py 4 0.25 0x0 > gpurun_out/ncu10.log 2>&1
python tools/sweep_batch.py 5 0.25 0x0 0x100 > gpurun_out/sweep10_b5.log 2>&1
cat gpurun_out/sweep10_b4.log gpurun_out/sweep10_b5.log
