#!/bin/bash
# learner + fusion evidence: the ncu launch list of one PPO update call (2 minibatches, C3 actor) and one
# `ncu --set full` capture each of the learner's tcgen05 GEMM and of the fused fusion kernel
OUT=gpurun_out/${1:-learner}
mkdir -p $OUT
CMD="python tools/bench_ppo.py --mb 2 --reps 1"
timeout 120 $CMD > $OUT/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --cache-control none --csv --log-file $OUT/launches_ppo.csv $CMD > $OUT/ncu_list.log 2>&1; echo "list exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 30 -c 2 -o $OUT/prof_gemm $CMD > $OUT/ncu_gemm.log 2>&1; echo "gemm exit $?"
timeout 120 python tools/bench_fuse.py > $OUT/fuse_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fuse_x -s 3 -c 1 -o $OUT/prof_fuse python tools/bench_fuse.py > $OUT/ncu_fuse.log 2>&1; echo "fuse exit $?"
