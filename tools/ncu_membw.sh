#!/bin/bash
# One `ncu --set full` capture of a membw_probe case's kernel:
#   tools/ncu_membw.sh "<case substring>" <kernel regex> <out name>
set -e
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k "regex:$2" -s 2 -c 1 -f \
    -o gpurun_out/$3 python tools/membw_probe.py --mb 256 --only "$1" > gpurun_out/$3.log 2>&1
ncu -i gpurun_out/$3.ncu-rep --page details --csv > gpurun_out/$3_details.csv
