#!/bin/bash
# compute-sanitizer passes over the round-2 kernels (cluster sq pass, streaming M-step, diet MAP kernel).
O=gpurun_out/${1:-r2san}; mkdir -p $O; export PYTHONPATH=$PWD
CS=compute-sanitizer
timeout 1500 $CS --tool memcheck --error-exitcode 9 python -m pytest -x -q tests/test_gpu_parity.py -k "not concurrent" > $O/memcheck_parity.log 2>&1; echo rc=$? >> $O/memcheck_parity.log
timeout 900 $CS --tool memcheck --error-exitcode 9 python -m pytest -x -q tests/test_gpu_steps.py tests/test_gpu_device_loop.py > $O/memcheck_steps.log 2>&1; echo rc=$? >> $O/memcheck_steps.log
timeout 1500 $CS --tool racecheck --error-exitcode 9 python -m pytest -x -q tests/test_gpu_parity.py -k "fixture_optimize or opt_in or stream" > $O/racecheck.log 2>&1; echo rc=$? >> $O/racecheck.log
timeout 1200 $CS --tool synccheck --error-exitcode 9 python -m pytest -x -q tests/test_gpu_parity.py -k "fixture_optimize or opt_in or stream" > $O/synccheck.log 2>&1; echo rc=$? >> $O/synccheck.log
timeout 600 $CS --tool memcheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > $O/memcheck_smoke.log 2>&1; echo rc=$? >> $O/memcheck_smoke.log
echo done > $O/done
