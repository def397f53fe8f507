# chunked visibility raster: parity (forced on for small meshes), C4 stage
# times with the dense and the sparse blend, and 16x16 sort tiles
set -x
timeout 900 python -m pytest tests/test_gpu_scale.py -q -m gpu -k "binned or c4" > gpurun_out/c4b_tests.log 2>&1
echo "tests rc=$?"
python profiles/profile_frames.py --config c4 --warm 20 --frames 6 --timing --trace > gpurun_out/c4b_dense.txt 2>&1
VMSPLAT_BLEND_SPARSE=1 python profiles/profile_frames.py --config c4 --warm 20 --frames 6 --timing --trace > gpurun_out/c4b_sparse.txt 2>&1
VMSPLAT_TILE=16 python profiles/profile_frames.py --config c4 --warm 20 --frames 6 --timing --trace > gpurun_out/c4b_t16.txt 2>&1
rm -rf /dev/shm/vmsplat_bench /dev/shm/vmsplat_test_c4
tail -3 gpurun_out/c4b_tests.log
grep -E "^2[0-5] |blend:|p100" gpurun_out/c4b_dense.txt gpurun_out/c4b_sparse.txt gpurun_out/c4b_t16.txt | cut -c1-330
