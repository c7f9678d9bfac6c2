set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g35_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
for kr in 0 1024 2048 4096; do echo "KR $kr: $(IHT_ADJ_KR=$kr timeout 120 python scripts/prof_parts.py c2 2>&1 | grep adjoint)"; done > $OUT/g35_probe.log
echo done
