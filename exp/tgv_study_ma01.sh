#!/bin/bash
# TGV Ma 0.1, Re 1600 (BASELINE configs[1]) resolution ladder to t = 10: CGKS-5th and GKS-2nd
D=gpurun_out/tgv_study
mkdir -p $D
run() { timeout 1500 python tools/tgv_history.py --case tgv --n $2 --scheme $1 --t-end 10 --every $3 > $D/hist_$1_$2.jsonl 2> $D/err_$1_$2.log; echo "$1 $2 rc $?"; }
run cgks5 64 40
run cgks5 96 60
run cgks5 128 80
run gks2 128 50
run gks2 192 75
run gks2 256 100
run cgks5 192 120
