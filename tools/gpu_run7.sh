mkdir -p gpurun_out
python -m pytest tests/test_fuzz.py tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider -k "not full" > gpurun_out/pytest7.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest7.log
tail -3 gpurun_out/pytest7.log
bash tools/gpu_run6.sh
