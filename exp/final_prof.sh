#!/bin/bash
# round-end measurement pass: bench line, ncu launch list, one --set full capture of a stage
V=${1:-v18}
python bench.py > gpurun_out/${V}_bench.log 2>&1; echo "bench rc $?"
tail -1 gpurun_out/${V}_bench.log > gpurun_out/${V}_bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${V}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${V}_ncu_l.log 2>&1; echo "ncu list rc $?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_flux|k_recon5|k_update" -s 10 -c 5 \
  -o gpurun_out/${V}_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${V}_ncu_f.log 2>&1; echo "ncu full rc $?"
ls -la gpurun_out/ | grep ${V}
