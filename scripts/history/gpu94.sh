set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g94_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
bash scripts/gpu_sweep.sh r01f
bash scripts/gpu_profiles.sh r01f
timeout 1000 python -m pytest tests -m gpu -x -q --timeout 300 > $OUT/r01f_tests.log 2>&1; echo "tests rc=$?" >> $OUT/r01f_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/r01f_smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/r01f_smoke.log
echo done
