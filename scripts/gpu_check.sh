timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/gputests.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
