mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_fuzz.py -x -q -m gpu -p no:cacheprovider -k "not full" > gpurun_out/pytest11.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest11.log
tail -3 gpurun_out/pytest11.log
python tools/sweep_decode.py 0x0 0x400000 > gpurun_out/sweep11_dec2.log 2>&1
cat gpurun_out/sweep11_dec2.log
