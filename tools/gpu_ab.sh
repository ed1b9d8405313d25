# A/B: for each lib variant under paper_1709_08990_b200/lib/var*/: batch GPU tests, then the cfg4 sweep.
# Usage: bash tools/gpu_ab.sh TAG FLAGS...
T=$1; shift
mkdir -p gpurun_out
for V in paper_1709_08990_b200/lib/var*/; do
  v=$(basename $V); cp $V/libbytecodec_b200.so paper_1709_08990_b200/lib/
  echo "== $v" >> gpurun_out/ab_$T.log
  timeout 600 python -m pytest tests/test_batch_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2 >> gpurun_out/ab_$T.log
  timeout 300 python tools/sweep_batch.py 4 1.0 "$@" >> gpurun_out/ab_$T.log 2>&1
done
cat gpurun_out/ab_$T.log
