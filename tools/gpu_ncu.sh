#!/bin/bash
# ncu passes: launch lists of one step (B, D) and full captures of the dominant kernels.
TAG=${1:-r2ncu}; O=gpurun_out/$TAG; mkdir -p $O; export PYTHONPATH=$PWD
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
timeout 600 ncu $M --log-file $O/launches_B.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launch_B.log 2>&1
timeout 900 ncu $M --log-file $O/launches_D.csv python bench.py --config D --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launch_D.log 2>&1
F="--set full --clock-control none --import-source on"
timeout 900 ncu $F -k regex:k_map_fused -s 60 -c 1 -o $O/full_B python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_full_B.log 2>&1
timeout 900 ncu $F -k regex:"k_fold_sum_ldg|k_fold_sq_cluster" -s 8 -c 2 -o $O/full_B_mstep python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_full_B_mstep.log 2>&1
timeout 900 ncu $F -k regex:k_map_fused -s 30 -c 1 -o $O/full_D python bench.py --config D --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_full_D.log 2>&1
timeout 900 ncu $F -k regex:"k_mstep_stream|k_label_scatter_warp" -s 4 -c 2 -o $O/full_D_mstep python bench.py --config D --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_full_D_mstep.log 2>&1
echo done > $O/done
