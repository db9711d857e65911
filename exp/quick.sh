#!/bin/bash
# quick perf comparison of library variants (TGV 128^3 CGKS-5th)
for lib in "$@"; do
  CGKS_LIB=$lib python bench.py --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/q.log 2>&1
  tail -1 gpurun_out/q.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step'],2), {k:round(v['ms_per_launch'],3) for k,v in d['per_kernel'].items() if v['ms_per_launch']>0.1})" || tail -5 gpurun_out/q.log
done
