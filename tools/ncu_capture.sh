#!/bin/bash
# One `ncu --set full` capture of one kernel launch during the full-schedule
# Shadow/drill run (dev tool, run on the GPU box):
#   tools/ncu_capture.sh KERNEL_REGEX SKIP NAME  ->  gpurun_out/NAME.ncu-rep
cd "$(dirname "$0")/.."
ncu --set full --import-source on --clock-control none -k "regex:$1" -s "$2" -c 1 -o "gpurun_out/$3" \
  python tools/prof_run.py 4096 300 100 100 > "gpurun_out/$3.log" 2>&1
