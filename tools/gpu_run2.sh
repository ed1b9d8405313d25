mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest2.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench2.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench2.log
python tools/sweep_encode.py 3 0x0 0x1000 > gpurun_out/sweep_enc3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"svb_encode_tile|svb_size_scan" -s 4 -c 2 -o gpurun_out/enc3_tile python tools/sweep_encode.py 3 0x0 > gpurun_out/ncu_enc3_tile.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"svb_encode1" -s 2 -c 1 -o gpurun_out/enc3_one python tools/sweep_encode.py 3 0x1000 > gpurun_out/ncu_enc3_one.log 2>&1
tail -3 gpurun_out/pytest2.log; tail -c 600 gpurun_out/bench2.log; cat gpurun_out/sweep_enc3.log
