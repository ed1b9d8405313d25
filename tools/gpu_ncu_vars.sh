# ncu --set full of the cfg4 x0.25 batch decode for each lib variant under paper_1709_08990_b200/lib/var*/.
# Usage: bash tools/gpu_ncu_vars.sh TAG [REGEX]
T=$1; RX=${2:-svb_decode_batch3}
mkdir -p gpurun_out
for V in paper_1709_08990_b200/lib/var*/; do
  v=$(basename $V); cp $V/libbytecodec_b200.so paper_1709_08990_b200/lib/
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$RX" -s 2 -c 1 \
    -o gpurun_out/ncu_${T}_$v python tools/sweep_batch.py 4 0.25 0x0 > gpurun_out/ncu_${T}_$v.log 2>&1
  tail -1 gpurun_out/ncu_${T}_$v.log
done
