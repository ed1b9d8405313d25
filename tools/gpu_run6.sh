mkdir -p gpurun_out
python tools/sweep_encode.py 3 0x0 0x1000 > gpurun_out/sweep6_enc3.log 2>&1
python tools/sweep_encode.py 2 0x0 > gpurun_out/sweep6_enc2.log 2>&1
python tools/trace_encode1.py 3 0x1000 > gpurun_out/trace6_cfg3.log 2>&1
cat gpurun_out/sweep6_enc3.log gpurun_out/sweep6_enc2.log gpurun_out/trace6_cfg3.log
