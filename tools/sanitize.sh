#!/bin/bash
# compute-sanitizer passes over tools/sanitize.py (one tool per pass).  Usage: bash tools/sanitize.sh TAG
set -u
R=${1:-x}
O=gpurun_out/r02
mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool memcheck --leak-check no --error-exitcode 9 python tools/sanitize.py > $O/san_memcheck_${R}.log 2>&1; echo "memcheck rc=$?"
timeout 1200 $CS --tool racecheck --racecheck-report analysis --error-exitcode 9 python tools/sanitize.py --quick > $O/san_racecheck_${R}.log 2>&1; echo "racecheck rc=$?"
timeout 900 $CS --tool synccheck --error-exitcode 9 python tools/sanitize.py --quick > $O/san_synccheck_${R}.log 2>&1; echo "synccheck rc=$?"
timeout 900 $CS --tool initcheck --error-exitcode 9 python tools/sanitize.py --quick > $O/san_initcheck_${R}.log 2>&1; echo "initcheck rc=$?"
