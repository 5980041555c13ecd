#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
tools/r2_call.sh r2e k_project
tools/r2_deflate.sh r2e
