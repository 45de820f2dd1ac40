#!/bin/bash
# A/B of k_mstep_stream variants (build/variants/*.so) at config D: the
# D-shape parity tests per variant, then bench lines (tools/ab.sh).
#   bash tools/ab_mstep.sh OUTDIR variant...
export PYTHONPATH=$PWD
O=$1; shift; mkdir -p $O
for v in "$@"; do
  DPMRF_CUDA_LIB=build/variants/$v.so timeout 300 python -m pytest tests/test_gpu_bench_shapes.py -q -x -m gpu 2>&1 | tail -1 | sed "s/^/$v parity: /" >> $O/parity.txt
done
ROUNDS=${ROUNDS:-2} bash tools/ab.sh $O "D" "$@" > /dev/null 2>&1
cat $O/parity.txt; sort $O/summary.txt
for f in $O/*.D.1.jsonl; do python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d['kernel_ms_per_step']['mstep_us_per_em'],1))" $f; done
