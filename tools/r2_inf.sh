#!/bin/bash
# decode-side parity + timing
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/$1; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "inflate or decompress or zlib or decode" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python tools/dec_prof.py > $O/dec.log 2>&1
for i in 1 2; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/b_$i.log 2>&1; done
