# Full measurement pass (one gpurun call): GPU tests, smoke, bench (all configs), the CPU
# reference arm, a cold launch list of the headline step and one ncu --set full of the
# dominant kernel.  Usage: bash tools/gpu_full.sh TAG
T=${1:-vX}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$T.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$T.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$T.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$T.log
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/ref_$T.log 2>&1; echo "ref rc=$?" >> gpurun_out/ref_$T.log
for W in cfg3 cfg2 cfg4 cfg5; do
  python bench.py --workload $W --no-cpu --no-e2e --steps 2 --warmup 3 > gpurun_out/plain_$W.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/launches_${T}_$W.csv python bench.py --workload $W --no-cpu --no-e2e --steps 2 --warmup 3 > /dev/null 2>&1
done
python tools/sweep_encode.py 3 0x0 > gpurun_out/sweep_$T.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"svb_encode1" -s 2 -c 1 -o gpurun_out/ncu_${T}_cfg3enc python tools/sweep_encode.py 3 0x0 > /dev/null 2>&1
for f in gpurun_out/pytest_$T.log gpurun_out/smoke_$T.log; do tail -n 2 $f; done; grep "\[bench\]" gpurun_out/bench_$T.log | cut -c 1-400; tail -c 300 gpurun_out/ref_$T.log
bash tools/gpu_ncu_batch.sh ${T}b 0x0 > /dev/null 2>&1
