# build the committed HEAD's library into .ab/ (for scripts/gpu_ab.sh)
set -e
git stash -q
python -c "from paper_2506_19415_b200 import build as b; b.build()" > /dev/null
mkdir -p .ab && cp paper_2506_19415_b200/libvmsplat_b200.so .ab/libvmsplat_b200_old.so
git stash pop -q
python -c "from paper_2506_19415_b200 import build as b; b.build()" > /dev/null
