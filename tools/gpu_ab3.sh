# A/B of the cfg3 encode over lib variants under paper_1709_08990_b200/lib/var*/.  Usage: bash tools/gpu_ab3.sh TAG [CFG]
T=$1; C=${2:-3}
mkdir -p gpurun_out
for V in paper_1709_08990_b200/lib/var*/; do
  v=$(basename $V); cp $V/libbytecodec_b200.so paper_1709_08990_b200/lib/
  echo "== $v" >> gpurun_out/ab3_$T.log
  timeout 300 python tools/sweep_encode.py $C 0x0 0x0 >> gpurun_out/ab3_$T.log 2>&1
done
cat gpurun_out/ab3_$T.log
