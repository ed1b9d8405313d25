# cfg5 (and cfg4) batch timings over lib variants under paper_1709_08990_b200/lib/var*/.  Usage: bash tools/gpu_ab5.sh TAG
T=$1
mkdir -p gpurun_out
for V in paper_1709_08990_b200/lib/var*/; do
  v=$(basename $V); cp $V/libbytecodec_b200.so paper_1709_08990_b200/lib/
  echo "== $v" >> gpurun_out/ab5_$T.log
  timeout 300 python tools/sweep_batch.py 5 1.0 0x0 >> gpurun_out/ab5_$T.log 2>&1
  timeout 300 python tools/sweep_batch.py 4 1.0 0x0 >> gpurun_out/ab5_$T.log 2>&1
done
cat gpurun_out/ab5_$T.log
