#!/bin/bash
# ncu --set full of one adjoint launch of the config-4 bench (plain run first, as the recipe requires)
TAG=${1:-prof}; shift || true
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e $*"
$CMD > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err && \
ncu --set full --clock-control none --import-source on -k regex:adjoint_mma -s 3 -c 1 -o gpurun_out/${TAG}_adjoint $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo "rc=$?"
