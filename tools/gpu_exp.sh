# Experiment pass: for the current build, or for every library variant under
# paper_1709_08990_b200/lib/var_*/ in turn: codec GPU tests (skipped with "notest"), then the
# cfg3 / cfg2 encode sweeps and the cfg4 / cfg5 batch sweeps.  Usage: bash tools/gpu_exp.sh TAG [notest]
T=$1
L=paper_1709_08990_b200/lib
mkdir -p gpurun_out
run() {
  if [ "$2" != "notest" ]; then
    timeout 1200 python -m pytest tests/test_batch_gpu.py tests/test_fuzz.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "not full" > gpurun_out/x_${T}_$1.log 2>&1; tail -n 2 gpurun_out/x_${T}_$1.log
  fi
  (timeout 300 python tools/sweep_encode.py 3 0x0; timeout 300 python tools/sweep_encode.py 2 0x0; timeout 300 python tools/sweep_batch.py 4 1.0 0x0; timeout 300 python tools/sweep_batch.py 5 1.0 0x0) 2>&1 | tee -a gpurun_out/x_${T}_$1.log
}
if ls -d $L/var_*/ > /dev/null 2>&1; then
  for V in $L/var_*/; do v=$(basename $V); cp $V/libbytecodec_b200.so $L/; echo "== $v"; run $v $2; done
else
  run cur $2
fi
