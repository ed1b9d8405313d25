mkdir -p gpurun_out
python tools/trace_encode1.py 3 0x1000 > gpurun_out/trace_e1_cfg3.log 2>&1
python tools/trace_encode1.py 2 > gpurun_out/trace_e1_cfg2.log 2>&1
cat gpurun_out/trace_e1_cfg3.log gpurun_out/trace_e1_cfg2.log
bash tools/gpu_run4.sh
