#!/bin/bash
# ncu passes at config D: launch list of one step, full captures of the fused MAP kernel and the M-step folds.
TAG=${1:-r2h}; O=gpurun_out/$TAG; mkdir -p $O; export PYTHONPATH=$PWD
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_D.csv \
   python bench.py --config D --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launch_D.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_map_fused -s 30 -c 1 \
   -o $O/full_D python bench.py --config D --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_full_D.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fold|k_tile|k_label" -s 6 -c 6 \
   -o $O/full_D_mstep python bench.py --config D --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_full_D_mstep.log 2>&1
DPMRF_CUDA_LIB=build/variants/probe.so timeout 300 python tools/mstep_probe.py D 2 > $O/probe_D.jsonl 2> $O/probe_D.err
echo done > $O/done
