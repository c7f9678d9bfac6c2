#!/bin/bash
# RecoveryReport (iht_solver_report) parity tests
OUT=gpurun_out/r02g60; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_report.py -m gpu -q -x -rf -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
