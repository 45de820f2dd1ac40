#!/bin/bash
# Full GPU pass: tests, smoke, bench lines of every config, reference arm.
TAG=${1:-r2q}; O=gpurun_out/$TAG; mkdir -p $O; export PYTHONPATH=$PWD
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
nproc > $O/nproc.txt; lscpu | grep "Model name" >> $O/nproc.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_B.jsonl 2> $O/bench_B.err
timeout 300 python bench.py --config A > $O/bench_A.jsonl 2> $O/bench_A.err
timeout 600 python bench.py --config C --cpu-seconds 20 > $O/bench_C.jsonl 2> $O/bench_C.err
timeout 900 python bench.py --config D --steps 5 > $O/bench_D.jsonl 2> $O/bench_D.err
timeout 900 python bench.py --config D --steps 3 --local-parts 2 > $O/bench_D_local2.jsonl 2> $O/bench_D_local2.err
timeout 600 python bench.py --config E --slices 64 --steps 3 > $O/bench_E64.jsonl 2> $O/bench_E64.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_B.jsonl 2> $O/bench_ref_B.err
echo done > $O/done
