set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g24_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/g24_smi.txt 2>&1
bash scripts/gpu_sweep.sh r01b
bash scripts/gpu_profiles.sh r01b
echo done
