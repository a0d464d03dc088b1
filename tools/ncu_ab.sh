# ncu --set full (source-level) capture of one K_A/K_B blur launch of tools/blur_ab.py's driver:
#   bash tools/ncu_ab.sh TAG [LIB]    -> gpurun_out/TAG.ncu-rep  (LIB: an A/B build, default in-tree)
TAG=${1:-blur}
if [ -n "$2" ]; then export MLSQR_LIB_PATH=$(readlink -f "$2"); fi
timeout 600 ncu --set full --import-source on --clock-control none -k regex:blur3d_mma -s 30 -c 1 \
  -o gpurun_out/${TAG} python tools/blur_ab.py --child > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu $TAG rc=$?"
