# compute-sanitizer on the round-2 kernels: device page table (dpt_update_k,
# chunk kernels), LOD (lod_seed_k, lod_lloyd_k), certified blend + repair
O=gpurun_out/r2/sanitize2; mkdir -p $O
CS="compute-sanitizer --print-limit 50 --error-exitcode 9"
timeout 1500 $CS --tool memcheck python -m pytest tests/test_gpu_dpt.py -m gpu -q -x -k "reference_traces or unit_cases or pipelined" > $O/dpt_memcheck.log 2>&1; echo "dpt memcheck rc=$?"
timeout 1500 $CS --tool racecheck python -m pytest tests/test_gpu_dpt.py -m gpu -q -x -k "unit_cases" > $O/dpt_racecheck.log 2>&1; echo "dpt racecheck rc=$?"
timeout 1500 $CS --tool memcheck python -m pytest tests/test_lod.py -m gpu -q -x -k "cluster_page_matches or merge_cluster_matches or ref_pyramid" > $O/lod_memcheck.log 2>&1; echo "lod memcheck rc=$?"
timeout 1500 $CS --tool racecheck python -m pytest tests/test_lod.py -m gpu -q -x -k "cluster_page_matches" > $O/lod_racecheck.log 2>&1; echo "lod racecheck rc=$?"
timeout 1500 $CS --tool memcheck python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "certified_repair or certified_blend_banded" > $O/cert_memcheck.log 2>&1; echo "cert memcheck rc=$?"
tail -n 3 $O/*.log
