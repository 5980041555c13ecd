#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
tools/r2_call.sh r2i "k_project"
tools/r2_sweep.sh r2i "MLK_PROJECT_OVERLAP=0" "MLK_PROJECT_OVERLAP=1"
