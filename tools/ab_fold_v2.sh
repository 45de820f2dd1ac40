export PYTHONPATH=$PWD
O=gpurun_out/abv2; mkdir -p $O
DPMRF_CUDA_LIB=build/variants/v2on.so timeout 600 python -m pytest tests/test_gpu_bench_shapes.py tests/test_gpu_parity.py tests/test_gpu_steps.py -q -x -m gpu 2>&1 | tail -1 > $O/parity.txt
ROUNDS=2 bash tools/ab.sh $O "B C D" v2off v2on > /dev/null 2>&1
cat $O/parity.txt; sort $O/summary.txt
for f in $O/*.1.jsonl; do python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1].split('/')[-1], round(d['kernel_ms_per_step']['mstep_us_per_em'],2))" $f; done
