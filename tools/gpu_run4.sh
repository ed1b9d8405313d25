mkdir -p gpurun_out
python tools/sweep_batch.py 4 0.25 0x0 > gpurun_out/sweep4_b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"batch3" -s 2 -c 2 -o gpurun_out/b3_cfg4 python tools/sweep_batch.py 4 0.25 0x0 > gpurun_out/ncu4.log 2>&1
cat gpurun_out/sweep4_b.log; tail -2 gpurun_out/ncu4.log
