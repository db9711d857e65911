#!/bin/bash
# A/B of two libraries on TGV 128^3 (default) and the high-speed TGV 116^3
for lib in "$@"; do
  for wl in tgv128 tgv_ss116; do
    CGKS_LIB=$lib python bench.py --workload $wl --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>&1
    tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib $wl', round(d['ms_per_step'],3), {k:round(v['ms_per_launch'],3) for k,v in d['per_kernel'].items() if v['ms_per_launch']>0.1})" || tail -3 gpurun_out/ab.log
  done
done
