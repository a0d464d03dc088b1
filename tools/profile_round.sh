#!/bin/bash
# Round measurement recipe (run on the GPU box via gpurun):  bash tools/profile_round.sh TAG
#   bench line (+ CPU baseline, e2e), reference arm, ncu launch list of the bench (with DRAM bytes),
#   one `ncu --set full` capture per hot kernel, and one bench line per other BASELINE config.
#   Outputs land in gpurun_out/TAG_*.
TAG=${1:-r}
O=gpurun_out
mkdir -p $O
timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; echo "bench rc=$?"
tail -1 $O/${TAG}_bench.json
timeout 900 python bench.py --impl reference > $O/${TAG}_ref.json 2> $O/${TAG}_ref.err; echo "ref rc=$?"
tail -1 $O/${TAG}_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 700 --csv --log-file $O/${TAG}_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
  > $O/${TAG}_ncu_launch.log 2>&1; echo "launch list rc=$?"
# one full capture per hot kernel, aimed at a level-0 launch of the 512^3 driver:
#   blur: 6th launch (mlsqr iteration 1's K_A, with the xpby/norm epilogue); the V-cycle kernels: every
#   launch of the driver's 2nd V-cycle (all levels), of which summarize.py keeps the longest; update: first.
# (gpurun brings back at most 64 MiB: only the single-launch C5 captures carry the SASS/source pages)
cap() {  # name regex skip count   (summarize.py keeps the longest captured launch = level 0)
  local src="--import-source on"; [ "${4:-1}" != 1 ] && src=""
  timeout 600 ncu --set full --clock-control none $src --kernel-name-base demangled \
    -k "regex:$2" -s $3 -c ${4:-1} -o $O/${TAG}_full_$1 python profiles/kernel_driver.py --reps 2 --iters 2 \
    > $O/${TAG}_full_$1.log 2>&1; echo "full $1 rc=$?"
}
cap blur 'blur3d_(mma|pipe)' 5
cap sweep_fn 'sweep_fn(_tma)?_kernel' 4 4
cap sweep_prolong 'sweep_zm_kernel<.int.3, .int.2' 4 4
cap sweep_normal 'sweep_zm_kernel<.int.3, .int.1' 7 7
cap restrict 'restrict_zm_kernel' 4 4
cap update 'update_kernel' 0
# the other BASELINE configs (parity configs; one bench line each, no CPU baseline; enough steps for
# the clock sampler to see the timed region)
declare -A STEPS=([c1]=300 [c2]=200 [c3]=100 [c4]=5)
for c in c1 c2 c3 c4; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --steps ${STEPS[$c]} --warmup 3 > $O/${TAG}_bench_$c.json 2> $O/${TAG}_bench_$c.err
  echo "bench $c rc=$?"
done
# one full capture per hot kernel of the small / dense configs (C2 2D blur + fused first sweeps, C3 128^3 blur,
# C4 dense A x / A^T y), aimed at launches inside the first timed outer step
capc() {  # name config regex skip
  timeout 600 ncu --set full --clock-control none --kernel-name-base demangled \
    -k "regex:$3" -s $4 -c 1 -o $O/${TAG}_full_$1 python bench.py --config $2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
    > $O/${TAG}_full_$1.log 2>&1; echo "full $1 rc=$?"
}
capc c2_blur2d c2 'blur2d_reg_kernel' 40
capc c2_sweep_fn2d c2 'sweep_fn2d_kernel<.int.32' 20
capc c3_blur c3 'blur3d_(mma|pipe)' 40
capc c3_sweep_fn c3 'sweep_fn(_tma)?_kernel' 20
capc c4_gemv c4 'gemv_l1_(bulk_)?kernel' 10
capc c4_gemvt c4 'gemvt_kernel' 10
# summaries are made here, on the box (gpurun brings back at most 64 MiB): only the blur capture travels
python profiles/summarize.py launches $O/${TAG}_launches.csv $O/${TAG}_launches.md > /dev/null
python profiles/summarize.py dram_iter $O/${TAG}_launches.csv $O/${TAG}_dram_per_iter.json > /dev/null
: > $O/${TAG}_ncu_full.md
for k in blur sweep_fn sweep_prolong sweep_normal restrict update c2_blur2d c2_sweep_fn2d c3_blur c3_sweep_fn c4_gemv c4_gemvt; do
  python profiles/summarize.py full $O/${TAG}_full_$k.ncu-rep $O/_x.md > /dev/null 2>&1 && cat $O/_x.md >> $O/${TAG}_ncu_full.md
done
rm -f $O/_x.md
python profiles/summarize.py traffic $TAG $O/${TAG}_traffic.json > /dev/null
find $O -name '*.ncu-rep' ! -name "${TAG}_full_blur.ncu-rep" -delete
du -sh $O
