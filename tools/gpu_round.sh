#!/bin/bash
# One gpurun call: GPU tests, smoke, bench (+ reference arm), ncu launch list and --set full capture.
# Usage (from the repo root): gpurun --timeout 2400 -- 'bash tools/gpu_round.sh TAG [notests]'
TAG=${1:-run}
O=gpurun_out/$TAG
mkdir -p $O
if [ "$2" != "notests" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.txt 2>&1; echo "pytest rc=$?" >> $O/gpu_tests.txt
  tail -3 $O/gpu_tests.txt
fi
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; cat $O/bench.json
timeout 600 python bench.py --steps 100 --warmup 5 > $O/bench100.json 2> $O/bench100.err; echo "bench100 rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/ref.json 2> $O/ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_flux1|k_recon5|k_update' -s 10 -c 12 -o $O/full -f python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
ls -la $O
