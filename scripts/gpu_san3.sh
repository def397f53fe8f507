O=gpurun_out/r2/final2/sanitize; mkdir -p $O
CS="compute-sanitizer --print-limit 50 --error-exitcode 9"
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1   # writes the scene
( time timeout 2400 $CS --tool racecheck --kernel-regex kns=blend_k python profiles/profile_frames.py --warm 24 --frames 2 ) > $O/blend_racecheck.log 2>&1; echo "blend racecheck rc=$?"
tail -4 $O/blend_racecheck.log
( time timeout 1500 $CS --tool racecheck python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "session_matches_reference and True" ) > $O/session_racecheck.log 2>&1; echo "session racecheck rc=$?"
tail -4 $O/session_racecheck.log
