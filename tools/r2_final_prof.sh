#!/bin/bash
# round-2 evidence in one call: plain bench, launch list, ncu --set full of
# the top kernels (all ncu runs of a call count as one), decode-side kernels
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/$1
mkdir -p $O
ARGS="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks --no-train"
FULL="ncu --set full --clock-control none --import-source on"
python bench.py $ARGS > $O/plain.log 2>&1 && \
timeout 600 python tools/dec_prof.py > $O/dec_plain.log 2>&1 && {
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches.csv python bench.py $ARGS > $O/ncu_launches.log 2>&1
  timeout 900 $FULL -k regex:k_project -c 1 -o $O/project python bench.py $ARGS > $O/ncu_project.log 2>&1
  timeout 900 $FULL -k regex:k_deflate_warp -s 10 -c 2 -o $O/deflate python bench.py $ARGS > $O/ncu_deflate.log 2>&1
  timeout 900 $FULL -k regex:k_stage1 -c 1 -o $O/stage1 python bench.py $ARGS > $O/ncu_stage1.log 2>&1
  timeout 900 $FULL -k regex:k_kmeans -c 1 -o $O/kmeans python bench.py $ARGS > $O/ncu_kmeans.log 2>&1
  timeout 900 $FULL -k regex:k_probe_level -s 5 -c 1 -o $O/probe python bench.py $ARGS > $O/ncu_probe.log 2>&1
  timeout 900 $FULL -k regex:"k_inflate_warp|k_decode|k_varint" -c 3 -o $O/decode python tools/dec_prof.py > $O/ncu_decode.log 2>&1
}
echo "done rc=$?" >> $O/plain.log
