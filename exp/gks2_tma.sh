#!/bin/bash
# GKS-2nd flux with and without TMA staging (TGV 128^3)
python -m pytest tests -q -m gpu -x -k "gks2 or GKS2 or second" 2>&1 | tail -3
for v in 0 1; do
  if [ $v = 1 ]; then export CGKS_NO_TMA=1; fi
  python bench.py --scheme gks2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/g$v.log 2>&1
  tail -1 gpurun_out/g$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('notma=$v', round(d['ms_per_step'],3), {k:round(v['ms_per_launch'],3) for k,v in d['per_kernel'].items()})" || tail -5 gpurun_out/g$v.log
done
