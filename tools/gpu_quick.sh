O=gpurun_out/r2a; mkdir -p $O; export PYTHONPATH=$PWD
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
nproc > $O/nproc.txt; lscpu | grep "Model name" >> $O/nproc.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_B.jsonl 2> $O/bench_B.err
timeout 900 python bench.py --config D --steps 5 --no-cpu-baseline > $O/bench_D.jsonl 2> $O/bench_D.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_B.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launch_B.log 2>&1
echo done > $O/done
