mkdir -p gpurun_out
python tools/sweep_encode.py 3 0x0 > gpurun_out/sweep13.log 2>&1
python tools/sweep_encode.py 2 0x0 >> gpurun_out/sweep13.log 2>&1
python tools/sweep_decode.py 0x0 >> gpurun_out/sweep13.log 2>&1
python tools/sweep_batch.py 4 1.0 0x0 >> gpurun_out/sweep13.log 2>&1
python tools/sweep_batch.py 5 1.0 0x0 >> gpurun_out/sweep13.log 2>&1
cat gpurun_out/sweep13.log
python tools/sweep_encode.py 3 0x0 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"svb_encode1" -s 2 -c 1 -o gpurun_out/enc3_v4 python tools/sweep_encode.py 3 0x0 > /dev/null 2>&1
