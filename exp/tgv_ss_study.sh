#!/bin/bash
# equal-resolution study of the high-speed TGV (Table TGV-sup-4): CGKS-5th 116^3 and
# GKS-2nd 384^3 against a CGKS-5th 256^3 reference, to t = 10, one B200
mkdir -p gpurun_out/tgv_ss_study
T=${T_END:-10.0}
timeout 600 python tools/tgv_history.py --case tgv_ss --n 116 --scheme cgks5 --t-end $T --every 20 > gpurun_out/tgv_ss_study/hist_cgks5_116.jsonl 2> gpurun_out/tgv_ss_study/err_116.log; echo "116 rc $?"
timeout 900 python tools/tgv_history.py --case tgv_ss --n 384 --scheme gks2 --t-end $T --every 70 > gpurun_out/tgv_ss_study/hist_gks2_384.jsonl 2> gpurun_out/tgv_ss_study/err_384.log; echo "384 rc $?"
timeout 1200 python tools/tgv_history.py --case tgv_ss --n 256 --scheme cgks5 --t-end $T --every 45 > gpurun_out/tgv_ss_study/hist_cgks5_256.jsonl 2> gpurun_out/tgv_ss_study/err_256.log; echo "256 rc $?"
tail -1 gpurun_out/tgv_ss_study/*.jsonl
