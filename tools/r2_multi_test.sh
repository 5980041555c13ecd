#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/r2o
timeout 1500 python -m pytest tests/test_multi_gpu.py -m gpu -q -p no:cacheprovider > gpurun_out/r2o/multi_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2o/multi_tests.log
