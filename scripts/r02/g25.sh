#!/bin/bash
OUT=gpurun_out/r02g25; mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:thr_ -c 30 --csv python scripts/r02/c4_parts.py threshold > $OUT/ncu_thr.csv 2> $OUT/ncu.err
