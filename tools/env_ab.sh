#!/bin/bash
# Interleaved A/B of runtime switches on the bench configs.
#   VARIANTS="MLSQR_PDL=0;MLSQR_PDL=1" CONFIGS="c1 c2 c3" REPS=2 bash tools/env_ab.sh TAG
O=gpurun_out; T=${1:-ab}
declare -A STEPS=([c1]=300 [c2]=200 [c3]=100 [c4]=5 [c5]=3)
IFS=';' read -ra VS <<< "${VARIANTS:-MLSQR_PDL=0;MLSQR_PDL=1}"
for rep in $(seq 1 ${REPS:-2}); do
for c in ${CONFIGS:-c1 c2 c3}; do
  for v in "${VS[@]}"; do
    tag=$(echo "$v" | tr ' =/' '_-_' | tail -c 60)
    env $v timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps ${STEPS[$c]} --warmup 3 > $O/${T}_${c}_${tag}_r$rep.json 2>&1
    echo "$c [$v] rep=$rep rc=$? $(tail -1 $O/${T}_${c}_${tag}_r$rep.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); cr=d.get("class_rooflines") or {}; print(round(d["value"],1), d.get("clocks",{}).get("sm_mhz"), " ".join("%s=%.3f" % (k, v["ms_per_launch"]) for k, v in cr.items()))' 2>&1 | tail -1)"
  done
done
done
