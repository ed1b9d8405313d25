mkdir -p gpurun_out
python -m pytest tests/test_fuzz.py tests/test_gpu_parity.py tests/test_ctx_gpu.py -x -q -m gpu -p no:cacheprovider > gpurun_out/pytest3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest3.log
python tools/sweep_encode.py 3 0x0 0x1000 > gpurun_out/sweep3_enc3.log 2>&1
python tools/sweep_encode.py 2 0x0 > gpurun_out/sweep3_enc2.log 2>&1
python tools/sweep_encode.py 3 0x1000 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"svb_encode1" -s 2 -c 1 -o gpurun_out/enc3_one_v5 python tools/sweep_encode.py 3 0x1000 > gpurun_out/ncu3.log 2>&1
tail -3 gpurun_out/pytest3.log; cat gpurun_out/sweep3_enc3.log gpurun_out/sweep3_enc2.log
