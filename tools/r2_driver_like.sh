#!/bin/bash
# what the driver runs at round end (1 GPU): smoke, reference arm, own arm
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/$1
mkdir -p $O
( time python -c "import __graft_entry__ as g; g.smoke()" ) > $O/smoke.log 2>&1
( time python bench.py --impl reference ) > $O/ref.log 2>&1
( time python bench.py ) > $O/own.log 2>&1
