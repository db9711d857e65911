#!/bin/bash
# GPU-box check used during development: GPU test suite + a short bench summary line.
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['algorithmic_flops_per_cell_update'], {k:round(v['ms_per_launch'],3) for k,v in d['per_kernel'].items()})"
