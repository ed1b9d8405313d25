# ncu --set full of the cfg3 one-pass plain encode (svb_encode1_kernel).  Usage: bash tools/gpu_ncu_cfg3enc.sh TAG
T=$1
mkdir -p gpurun_out
python tools/sweep_encode.py 3 0x0 > gpurun_out/sweep3_$T.log 2>&1; cat gpurun_out/sweep3_$T.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"svb_encode1_kernel" -s 2 -c 1 \
  -o gpurun_out/ncu_${T}_cfg3enc python tools/sweep_encode.py 3 0x0 > gpurun_out/ncu3_$T.log 2>&1; tail -1 gpurun_out/ncu3_$T.log
