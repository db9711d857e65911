#!/bin/bash
echo "== graph"; timeout 600 python exp/crash_repro2.py 2>&1 | grep -v Warning | tail -6
echo "== graph, no TMA"; CGKS_NO_TMA=1 timeout 600 python exp/crash_repro2.py 2>&1 | grep -v Warning | tail -6
echo "== no graph"; CGKS_NO_GRAPH=1 timeout 600 python exp/crash_repro2.py 2>&1 | grep -v Warning | tail -6
