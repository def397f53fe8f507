# gpu parity tests + default bench (trace on: workspace/graph events to stderr)
set -x
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/gputests.log
VMSPLAT_TRACE=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1
tail -n 3 gpurun_out/gputests.log; grep -v Warn gpurun_out/bench.log | tail -c 2500
