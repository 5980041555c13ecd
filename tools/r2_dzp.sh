#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/r2r
timeout 600 python tools/deflate_prof.py > gpurun_out/r2r/deflate_prof.log 2>&1
