#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/r2et2
timeout 600 python tools/eb_trace.py > gpurun_out/r2et2/eb_trace_1.log 2>&1
