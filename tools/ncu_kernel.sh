#!/bin/bash
# One ncu --set full capture of kernel $1 (regex) from command "${@:2}" -> gpurun_out/$NAME.ncu-rep
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
K=$1; shift
ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-0} -c 1 -f -o gpurun_out/${NAME:-cap} "$@" > gpurun_out/${NAME:-cap}.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${NAME:-cap}.log
