#!/bin/bash
D=gpurun_out/chi_study
mkdir -p $D
for C in ${CHIS:-4 16}; do
  CGKS_LIB=exp/libcgks_chi$C.so timeout 600 python tools/tgv_history.py --case tgv_ss --n 116 --scheme cgks5 --t-end 10 --every 20 > $D/hist_cgks5_116_chiscale$C.jsonl 2> $D/err_$C.log; echo "C=$C rc $?"; tail -n 1 $D/err_$C.log
done
