set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g96_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
bash scripts/gpu_sweep.sh r01g
bash scripts/gpu_profiles.sh r01g
timeout 1000 python -m pytest tests -m gpu -x -q --timeout 300 > $OUT/r01g_tests.log 2>&1; echo "tests rc=$?" >> $OUT/r01g_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/r01g_smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/r01g_smoke.log
echo done
