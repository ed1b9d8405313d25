#!/bin/bash
# Dev tool: ncu --set full of the first launch matching a kernel regex.
# Usage: tools/ncu_kernel.sh NAME REGEX COUNT -- command...   (report: gpurun_out/NAME.ncu-rep)
name=$1; rx=$2; cnt=$3; shift 4
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$rx" -c "$cnt" -o "gpurun_out/$name" "$@" > "gpurun_out/$name.log" 2>&1
tail -2 "gpurun_out/$name.log"
