# r02 g73 (session 6): HEAD rebuilt in a fresh container; GPU tests, smoke, both bench arms
(timeout 1300 python -m pytest tests -m gpu -x -q 2>&1 | tail -8) > gpurun_out/g73_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/g73_smoke.log 2>&1
python bench.py > gpurun_out/g73_bench.json 2> gpurun_out/g73_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/g73_ref.json 2> gpurun_out/g73_ref.err
# r02 g74: ncu launch list of the config-4 bench at HEAD (a run under ncu is never a bench value)
mkdir -p gpurun_out/g74
timeout 500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -c 1500 --csv --log-file gpurun_out/g74/launches_c4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/g74/ncu.log 2>&1
python scripts/launch_summary.py gpurun_out/g74/launches_c4.csv > gpurun_out/g74/summary.txt
