set -x
python bench.py > gpurun_out/v19_cfg2_full.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/v19_reference.log 2>&1
python bench.py --workload cfg3 --no-cpu > gpurun_out/v19_cfg3.log 2>&1
python bench.py --workload cfg4 --no-cpu > gpurun_out/v19_cfg4.log 2>&1
python bench.py --workload cfg5 --no-cpu > gpurun_out/v19_cfg5.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:batch -c 8 --csv --log-file gpurun_out/v19_launches_cfg4.csv python bench.py --workload cfg4 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/v19_ncu4.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:batch -c 8 --csv --log-file gpurun_out/v19_launches_cfg5.csv python bench.py --workload cfg5 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/v19_ncu5.log 2>&1
