#!/bin/bash
# Repeated bench.py processes (config B) on one box: device value, e2e, the
# sorted per-call e2e wall times, the device time of the e2e calls, the
# upload alone and the active-set e2e -- to separate host/PCIe noise from
# device time.  Usage (on a GPU box): bash tools/bench_reps.sh [N]
mkdir -p gpurun_out/reps
show() { python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); e=d['e2e']
print(sys.argv[1], round(d['value']), round(e['value']), e['call_ms_sorted'][::3], round(e['device_ms_median'],3), round(e['upload_ms_median'],3), round(d['active_set']['e2e']))" $1; }
for i in $(seq 1 ${1:-2}); do
  python bench.py --no-cpu-baseline > gpurun_out/reps/b$i.log 2>&1; show gpurun_out/reps/b$i.log
done
