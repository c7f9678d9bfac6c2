set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/g37_build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
timeout 300 python scripts/prof_parts.py > $OUT/g37_parts.log 2>&1
for c in 1 2 3 5; do timeout 900 python bench.py --config $c --no-cpu-baseline --steps 5 > $OUT/g37_b$c.json 2> $OUT/g37_b$c.err; done
timeout 2400 python -m pytest tests -m gpu -x -q --timeout=600 > $OUT/g37_pytest.log 2>&1; echo "rc=$?" >> $OUT/g37_pytest.log
echo done
