#!/bin/bash
# final 1-GPU check: every GPU test, smoke, the reference arm and the own arm
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/$1; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
( time python -c "import __graft_entry__ as g; g.smoke()" ) > $O/smoke.log 2>&1
( time python bench.py --impl reference ) > $O/ref.log 2>&1
( time python bench.py ) > $O/own.log 2>&1
