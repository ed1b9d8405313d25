T=r2s3a
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$T.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$T.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$T.log
tail -3 gpurun_out/pytest_$T.log; grep "\[bench\]" gpurun_out/bench_$T.log | cut -c 1-400
