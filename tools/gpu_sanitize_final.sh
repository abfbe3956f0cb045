#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/sanitize_cases.py > gpurun_out/san_plain.log 2>&1; echo "plain rc=$?" >> gpurun_out/san_plain.log
bash tools/sanitize.sh
