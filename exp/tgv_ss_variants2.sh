#!/bin/bash
D=gpurun_out/tgv_ss_study
mkdir -p $D
for P in "tau_C=1" "relax_C=1" "tau_C=0"; do
  n=$(echo $P | tr '=' '_')
  timeout 600 python tools/tgv_history.py --case tgv_ss --n 116 --scheme cgks5 --param $P --t-end 10 --every 20 > $D/hist_cgks5_116_$n.jsonl 2> $D/err_$n.log; echo "$P rc $?"; tail -n 1 $D/err_$n.log
done
