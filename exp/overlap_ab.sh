#!/bin/bash
# z-slab path on one GPU (NCCL self halo) with and without the overlap, vs the plain context
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/o_plain.log 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --nccl-self > gpurun_out/o_ovl.log 2>&1
CGKS_NO_OVERLAP=1 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --nccl-self > gpurun_out/o_noovl.log 2>&1
for f in o_plain o_ovl o_noovl; do
  tail -1 gpurun_out/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', round(d['ms_per_step'],3), d['config']['parallelism'], d['gpu_launches'], {k:(round(v['ms_per_launch'],3), v['launches']) for k,v in d['per_kernel'].items()})" || tail -5 gpurun_out/$f.log
done
