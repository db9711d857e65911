#!/bin/bash
# A/B of library variants on one box: bash tools/ab.sh TAG steps lib1 lib2 ... (paths relative to the repo root; "base" = default)
TAG=$1; STEPS=$2; shift 2
O=gpurun_out/$TAG; mkdir -p $O
for rep in 1 2; do
for L in "$@"; do
  if [ "$L" = base ]; then unset CGKS_LIB; else export CGKS_LIB=$PWD/$L; fi
  n=$(basename $L .so)
  timeout 300 python bench.py --steps $STEPS --warmup 3 --no-cpu-baseline > $O/${n}_$rep.json 2> $O/${n}_$rep.err
  python - <<PY
import json
try:
    d=json.load(open("$O/${n}_$rep.json"))
    pk={k:round(v['ms_per_launch'],3) for k,v in d['per_kernel'].items() if k.startswith(('flux','recon','update'))}
    print("$n rep$rep", round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'], pk)
except Exception as e:
    print("$n rep$rep FAILED", e); print(open("$O/${n}_$rep.err").read()[-500:])
PY
done; done
