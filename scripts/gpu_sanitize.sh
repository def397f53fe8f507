# compute-sanitizer memcheck / racecheck / synccheck on smoke() and on three
# C2 frames (1080p, bench scene), logs under gpurun_out/sanitize/
mkdir -p gpurun_out/sanitize
cat > gpurun_out/sanitize/README <<X
compute-sanitizer on smoke() and on 3 C2 frames (bench scene)
X
CS="compute-sanitizer --print-limit 50 --error-exitcode 9"
SMOKE='import __graft_entry__ as g; g.smoke()'
for tool in memcheck racecheck synccheck; do
  timeout 1200 $CS --tool $tool python -c "$SMOKE" > gpurun_out/sanitize/smoke_$tool.log 2>&1
  echo "smoke $tool rc=$?"
done
for tool in memcheck racecheck; do
  timeout 1800 $CS --tool $tool python profiles/profile_frames.py --warm 2 --frames 1 > gpurun_out/sanitize/c2_$tool.log 2>&1
  echo "c2 $tool rc=$?"
done
VMSPLAT_VIS_BIN=1 timeout 1200 $CS --tool memcheck python profiles/profile_frames.py --warm 2 --frames 1 > gpurun_out/sanitize/c2_visbin_memcheck.log 2>&1
echo "c2 visbin memcheck rc=$?"
tail -4 gpurun_out/sanitize/*.log
