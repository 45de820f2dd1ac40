#!/bin/bash
# A/B timing of library variants built by tools/build_variant.sh:
#   bash tools/ab.sh OUTDIR "B D" base hoist ...      (runs on the GPU box)
# a variant "name:VAR=val" runs build/variants/name.so with VAR=val in the environment
O=$1; CFGS=$2; shift 2
mkdir -p $O
for round in $(seq 1 ${ROUNDS:-3}); do
for v in "$@"; do
  for c in $CFGS; do
    steps=10; [ "$c" = D ] && steps=5
    so=${v%%:*}; envs=""; [ "$so" != "$v" ] && envs=${v#*:}
    env $envs DPMRF_CUDA_LIB=build/variants/$so.so timeout 600 python bench.py --config $c --steps $steps \
      --no-cpu-baseline > $O/$v.$c.$round.jsonl 2> $O/$v.$c.$round.err
    python - "$O/$v.$c.$round.jsonl" "$v" "$c" <<'PY' | tee -a $O/summary.txt
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2], sys.argv[3], "value %.1f" % d["value"], "ms/step %.3f" % d["ms_per_step"],
          "frac %.3f" % d["roofline"]["frac"], "launch_us %.2f" % d["roofline"]["avg_launch_us"],
          "e2e %.1f" % d["e2e"]["value"])
except Exception as ex:
    print(sys.argv[2], sys.argv[3], "FAILED", ex)
PY
  done
done
done
