timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -2 > gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
