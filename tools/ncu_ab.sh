set -x
for v in base new; do
  if [ $v = base ]; then export MLSQR_LIB_PATH=$PWD/tools/ab_base.so; else unset MLSQR_LIB_PATH; fi
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:blur3d_mma -s 30 -c 1 -o gpurun_out/r2c_${v} python tools/blur_ab.py --child > gpurun_out/r2c_ncu_${v}.log 2>&1
  echo "$v rc=$?"
done
