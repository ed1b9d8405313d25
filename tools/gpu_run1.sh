set -x
nvidia-smi --query-gpu=name,memory.total --format=csv
nproc; free -g | head -2
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest1.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke1.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke1.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench1.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench1.log
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref1.log 2>&1; echo "ref rc=$?" >> gpurun_out/ref1.log
tail -3 gpurun_out/pytest1.log gpurun_out/smoke1.log; tail -c 1500 gpurun_out/bench1.log
