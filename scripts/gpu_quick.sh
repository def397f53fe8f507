timeout 1500 python -m pytest tests -m gpu -x -q -k "resolution or output_modes or overflow" 2>&1 | tail -30 > gpurun_out/gputests.log
