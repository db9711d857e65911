#!/bin/bash
D=gpurun_out/tgv_study
mkdir -p $D
timeout 1500 python tools/tgv_history.py --case tgv --n 296 --scheme gks2 --t-end 10 --every 115 > $D/hist_gks2_296.jsonl 2> $D/err_gks2_296.log; echo "gks2 296 rc $?"
timeout 900 python tools/tgv_history.py --case tgv --n 96 --scheme cgks5 --lines 1 --t-end 10 --every 60 > $D/hist_cgks5_96_lines.jsonl 2> $D/err_l96.log; echo "cgks5 96 lines rc $?"
