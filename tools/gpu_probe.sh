O=gpurun_out/r2b; mkdir -p $O; export PYTHONPATH=$PWD
DPMRF_CUDA_LIB=build/variants/probe.so timeout 300 python tools/mstep_probe.py B 3 > $O/probe_B.jsonl 2> $O/probe_B.err
DPMRF_CUDA_LIB=build/variants/probe.so timeout 300 python tools/mstep_probe.py D 2 > $O/probe_D.jsonl 2> $O/probe_D.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fold -s 20 -c 4 -o $O/full_B_fold python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_full_B_fold.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_map_fused -s 30 -c 1 -o $O/full_D python bench.py --config D --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_full_D.log 2>&1
