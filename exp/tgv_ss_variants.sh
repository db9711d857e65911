#!/bin/bash
# CGKS-5th 116^3 variants of the equal-resolution study (sensitivity of the under-resolved eps_S)
D=gpurun_out/tgv_ss_study
mkdir -p $D
timeout 600 python tools/tgv_history.py --case tgv_ss --n 116 --scheme cgks5 --nonlinear 0 --t-end 10 --every 20 > $D/hist_cgks5_116_linear.jsonl 2> $D/err_lin.log; echo "linear rc $?"; tail -n 2 $D/err_lin.log
timeout 600 python tools/tgv_history.py --case tgv_ss --n 116 --scheme cgks5 --chi-c 0.1 --t-end 10 --every 20 > $D/hist_cgks5_116_chi0.1.jsonl 2> $D/err_c1.log; echo "chi 0.1 rc $?"
timeout 600 python tools/tgv_history.py --case tgv_ss --n 116 --scheme cgks5 --chi-c 1.0 --t-end 10 --every 20 > $D/hist_cgks5_116_chi1.jsonl 2> $D/err_c2.log; echo "chi 1 rc $?"
timeout 900 python tools/tgv_history.py --case tgv_ss --n 116 --scheme cgks5 --lines 1 --t-end 10 --every 20 > $D/hist_cgks5_116_lines.jsonl 2> $D/err_l.log; echo "lines rc $?"; tail -n 2 $D/err_l.log
