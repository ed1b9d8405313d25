# Batch GPU tests + the cfg4 and cfg5 sweeps on the current build.  Usage: bash tools/gpu_quick.sh TAG
T=$1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_batch_gpu.py tests/test_fuzz.py -x -q -p no:cacheprovider > gpurun_out/q_$T.log 2>&1; tail -2 gpurun_out/q_$T.log
timeout 300 python tools/sweep_batch.py 4 1.0 0x0 0x0 2>&1 | tee -a gpurun_out/q_$T.log
timeout 300 python tools/sweep_batch.py 5 1.0 0x0 2>&1 | tee -a gpurun_out/q_$T.log
