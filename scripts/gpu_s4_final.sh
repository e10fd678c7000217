#!/bin/bash
# session-4 round evidence: lanes probe, full GPU suite, smoke, default bench (C4) with the driver's flags,
# C2 and C5 lines, reference arm, the bench launch list under ncu
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s4f}
timeout 2700 python -m pytest tests -x -q -m gpu --durations=15 > gpurun_out/${T}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log
cp gpurun_out/reference_suite_on_dropin.log gpurun_out/${T}_reference_suite.log 2>/dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench_c4.json 2> gpurun_out/${T}_bench_c4.err
echo "bench rc=$?" >> gpurun_out/${T}_bench_c4.err
timeout 900 python bench.py --config c2 > gpurun_out/${T}_bench_c2.json 2> gpurun_out/${T}_bench_c2.err
timeout 900 python bench.py --config c5 --no-extras > gpurun_out/${T}_bench_c5.json 2> gpurun_out/${T}_bench_c5.err
timeout 900 python bench.py --impl reference > gpurun_out/${T}_bench_ref_c4.json 2> gpurun_out/${T}_bench_ref_c4.err
B="python bench.py --steps 2 --warmup 1 --no-extras --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${T}_launches_c4.csv $B > gpurun_out/${T}_ncu_launch.log 2>&1
echo done
