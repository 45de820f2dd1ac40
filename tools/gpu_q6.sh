O=gpurun_out/r2k; mkdir -p $O; export PYTHONPATH=$PWD
DPMRF_CUDA_LIB=build/variants/probe.so timeout 300 python tools/stream_probe.py D 3 > $O/stream_probe_D.jsonl 2> $O/stream_probe_D.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_D.csv python bench.py --config D --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launch_D.log 2>&1
