#!/bin/bash
# One gpurun call: the bench line of every BASELINE configuration (both schemes) into gpurun_out/configs/
# (copied to profiles/r02/configs/).  Usage: gpurun --timeout 3000 -- 'bash tools/configs_round.sh'
O=gpurun_out/configs; mkdir -p $O
run() { n=$1; shift; timeout 1500 python bench.py "$@" > $O/$n.json 2> $O/$n.err; echo "$n rc=$?"; }
for s in cgks5 gks2; do
  run vortex40_$s --workload vortex40 --scheme $s --steps 20 --warmup 3
  run tgv64_$s --workload tgv64 --scheme $s --steps 20 --warmup 3
  run tgv128_$s --workload tgv128 --scheme $s --steps 20 --warmup 3
  run hit128_$s --workload hit128 --scheme $s --nonlinear 1 --steps 20 --warmup 3
  run shock_vortex_$s --workload shock_vortex --scheme $s --steps 20 --warmup 3
done
run tgv128_cgks5_lines --workload tgv128 --lines 1 --steps 20 --warmup 3
run tgv_ss116_cgks5 --workload tgv_ss116 --steps 20 --warmup 3
run tgv512slab_cgks5 --workload tgv512slab --steps 5 --warmup 3 --no-cpu-baseline
run tgv512_cgks5 --workload tgv512 --steps 3 --warmup 3 --no-cpu-baseline
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/configs/*.json")):
    try:
        d = [json.loads(l) for l in open(f) if l.startswith("{")][-1]
        print(f.split("/")[-1], round(d["ms_per_step"], 3), "%.3e" % d["value"], round(d["roofline"]["frac"], 3), round(d["roofline"]["step_frac"], 3),
              "%.3e" % d["e2e"]["value"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
    except Exception as e:
        print(f, "FAILED", e)
PY
