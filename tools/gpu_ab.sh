#!/bin/bash
# GPU pass: the whole -m gpu suite on the worktree build, then an A/B of variants.
#   bash tools/gpu_ab.sh TAG "B D" base v1 v2 ...
TAG=$1; CFGS=$2; shift 2
O=gpurun_out/$TAG; mkdir -p $O; export PYTHONPATH=$PWD
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
bash tools/ab.sh $O/ab "$CFGS" "$@"
echo done > $O/done
