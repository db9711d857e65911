#!/bin/bash
for lib in "$@"; do
  CGKS_LIB=$lib python bench.py --workload tgv512slab --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/abs.log 2>&1
  tail -1 gpurun_out/abs.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step'],2), {k:round(v['ms_per_launch'],2) for k,v in d['per_kernel'].items() if v['ms_per_launch']>0.5})" || tail -3 gpurun_out/abs.log
done
