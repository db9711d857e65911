#!/bin/bash
D=gpurun_out/crash
mkdir -p $D
CGKS_NO_GRAPH=1 CUDA_LAUNCH_BLOCKING=1 timeout 900 python tools/tgv_history.py --case tgv_ss --n 116 --scheme cgks5 --param tau_C=0 --t-end 3 --every 20 > $D/hist.jsonl 2> $D/err.log; echo "rc $?"; tail -n 3 $D/err.log; tail -n 2 $D/hist.jsonl
