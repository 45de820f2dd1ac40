#!/bin/bash
# One GPU-box pass: tests, smoke, bench lines, ncu launch list + full captures.
# usage: bash tools/gpu_round.sh [tag]
TAG=${1:-r1}
O=gpurun_out/$TAG
mkdir -p $O
export PYTHONPATH=$PWD
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
nproc > $O/nproc.txt; lscpu | grep "Model name" >> $O/nproc.txt
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_B.jsonl 2> $O/bench_B.err
timeout 300 python bench.py --config A > $O/bench_A.jsonl 2> $O/bench_A.err
timeout 600 python bench.py --config C --cpu-seconds 20 > $O/bench_C.jsonl 2> $O/bench_C.err
timeout 900 python bench.py --config D --steps 5 --no-cpu-baseline > $O/bench_D.jsonl 2> $O/bench_D.err
timeout 900 python bench.py --config D --steps 3 --local-parts 2 > $O/bench_D_local2.jsonl 2> $O/bench_D_local2.err
timeout 600 python bench.py --config E --slices 64 --steps 3 > $O/bench_E64.jsonl 2> $O/bench_E64.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_B.jsonl 2> $O/bench_ref_B.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_leaf_fold -s 2 -c 2 \
   -o $O/full_D_leaf python bench.py --config D --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_full_D_leaf.log 2>&1
timeout 900 python tools/bench_structure.py > $O/structure.jsonl 2> $O/structure.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_B.csv \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launch_B.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_D.csv \
   python bench.py --config D --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launch_D.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_map_fused -s 30 -c 2 \
   -o $O/full_D python bench.py --config D --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_full_D.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_map_fused -s 60 -c 2 \
   -o $O/full_B python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_full_B.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_leaf_fold -s 6 -c 2 \
   -o $O/full_B_leaf python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_full_B_leaf.log 2>&1
echo done > $O/done
