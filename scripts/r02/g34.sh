#!/bin/bash
OUT=gpurun_out/r02g34; mkdir -p $OUT
timeout 90 ./scripts/microbench/tc2_bench > $OUT/tc2.jsonl 2>&1; echo "rc=$?" >> $OUT/tc2.jsonl
