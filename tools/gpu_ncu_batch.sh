# ncu --set full of the cfg4 batch decode and encode kernels at x0.25 (one launch each).
# Usage: bash tools/gpu_ncu_batch.sh TAG [FLAGS]
T=${1:-vX}; F=${2:-0x0}
mkdir -p gpurun_out
python tools/sweep_batch.py 4 0.25 $F > gpurun_out/sweep_$T.log 2>&1; cat gpurun_out/sweep_$T.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"svb_(de|en)code_batch3" -s 4 -c 2 \
  -o gpurun_out/ncu_${T}_cfg4 python tools/sweep_batch.py 4 0.25 $F > gpurun_out/ncu_${T}.log 2>&1; tail -3 gpurun_out/ncu_${T}.log
