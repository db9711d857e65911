#!/bin/bash
# GENO chi scale (cgks_scheme.chi_scale) on the high-speed TGV 116^3 to t = 10
D=gpurun_out/chi_study
mkdir -p $D
for C in 4 8; do
  timeout 600 python tools/tgv_history.py --case tgv_ss --n 116 --scheme cgks5 --param chi_scale=$C --t-end 10 --every 20 > $D/hist_cgks5_116_chiscale$C.jsonl 2> $D/err_$C.log; echo "C=$C rc $?"
done
