#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/$1; mkdir -p $O
timeout 300 python tools/eb_trace.py > $O/eb.log 2>&1
