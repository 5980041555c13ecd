#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/$1
mkdir -p $O
timeout 600 python tools/kmeans_prof.py > $O/kmeans_prof.log 2>&1
