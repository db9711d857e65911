#!/bin/bash
D=gpurun_out/tgv_ss_study
mkdir -p $D
for N in 160 192; do
  timeout 900 python tools/tgv_history.py --case tgv_ss --n $N --scheme cgks5 --t-end 10 --every $((20 * N / 116)) > $D/hist_cgks5_$N.jsonl 2> $D/err_$N.log; echo "$N rc $?"
done
timeout 600 python tools/tgv_history.py --case tgv_ss --n 256 --scheme gks2 --t-end 10 --every 47 > $D/hist_gks2_256.jsonl 2> $D/err_g256.log; echo "gks2 256 rc $?"
