#!/bin/bash
# One GPU pass over the current tree: gpu tests, default bench line, the
# timed-region launch list, compute-sanitizer over tools/sanitize_run.py.
# usage (on the GPU box): bash tools/gpu_check.sh TAG [skip-tests] [skip-san]
tag=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_smi.txt 2>&1
if [ "$2" != "skip-tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x -rs > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc $?"
  tail -3 gpurun_out/${tag}_pytest.log
fi
timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc $?"
tail -c 600 gpurun_out/${tag}_bench.json
timeout 600 ncu --nvtx --nvtx-include timed/ --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras \
  > gpurun_out/${tag}_ncu_launch.log 2>&1; echo "ncu rc $?"
python tools/launch_summary.py gpurun_out/${tag}_launches.csv > gpurun_out/${tag}_launches.txt 2>&1
head -25 gpurun_out/${tag}_launches.txt
if [ "$3" != "skip-san" ]; then
  for tool in memcheck racecheck synccheck initcheck; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/${tag}_san_$tool.log 2>&1
    echo "sanitizer $tool rc $?"; tail -2 gpurun_out/${tag}_san_$tool.log
  done
fi
