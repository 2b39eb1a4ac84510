#!/bin/bash
mkdir -p gpurun_out
timeout 120 ./tools/microbench/green_probe > gpurun_out/green_probe.txt 2>&1; echo "rc=$?" >> gpurun_out/green_probe.txt
echo done
