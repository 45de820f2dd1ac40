O=gpurun_out/r2e; mkdir -p $O; export PYTHONPATH=$PWD
DPMRF_CUDA_LIB=build/variants/probe.so timeout 300 python tools/mstep_probe.py B 3 > $O/probe_B.jsonl 2> $O/probe_B.err
bash tools/gpu_ab.sh r2e "B" diet3 diet3:DPMRF_CLUSTER_SQ=0
