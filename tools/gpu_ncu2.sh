# ncu --set full of the cfg3 one-pass encode and of the cfg4 batch kernels (x0.25).  Usage: bash tools/gpu_ncu2.sh TAG
T=$1
mkdir -p gpurun_out
python tools/sweep_encode.py 3 0x0 > gpurun_out/sweep_$T.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"svb_encode1" -s 2 -c 1 -o gpurun_out/ncu_${T}_cfg3enc python tools/sweep_encode.py 3 0x0 > /dev/null 2>&1
bash tools/gpu_ncu_batch.sh ${T}b 0x0 > /dev/null 2>&1
cat gpurun_out/sweep_$T.log gpurun_out/sweep_${T}b.log
