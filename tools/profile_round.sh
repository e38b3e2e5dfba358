#!/bin/bash
# One GPU call per round: benches (C3 default with cpu_baseline + e2e, C2, C4, C5, the reference arm), the ncu
# launch lists of a C3 run (fused rollout kernel, and POD_FUSED=0: the separate launches) with the L2 left warm
# between launches (--cache-control none: DRAM reads AND write-backs land in a steady multi-launch window,
# averaged per launch), one `ncu --set full` capture per hot kernel, the learner / fusion micro-benches, the
# per-phase clock64 traces and the fused kernel's per-step phases (globaltimer build).
# Outputs under gpurun_out/$1/ (scratch; summaries are copied to profiles/ by tools/summarize_ncu.py).
OUT=gpurun_out/${1:-prof}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt
timeout 900 python bench.py > $OUT/bench_c3.json 2> $OUT/bench_c3.err; echo "C3 exit $?"
timeout 600 python bench.py --config C2 > $OUT/bench_c2.json 2> $OUT/bench_c2.err; echo "C2 exit $?"
timeout 600 python bench.py --config C4 --no-cpu-baseline > $OUT/bench_c4.json 2> $OUT/bench_c4.err; echo "C4 exit $?"
timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "C5 exit $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "REF exit $?"
timeout 300 python tools/bench_ppo.py > $OUT/ppo_bench_1.json 2> $OUT/ppo_bench.err; echo "ppo1 exit $?"
timeout 300 python tools/bench_ppo.py --pods 8 > $OUT/ppo_bench_8.json 2>> $OUT/ppo_bench.err; echo "ppo8 exit $?"
timeout 300 python tools/bench_fuse.py > $OUT/fuse_bench.json 2> $OUT/fuse_bench.err; echo "fuse exit $?"
POD_FUSED=0 timeout 300 python tools_trace.py C3 60 > $OUT/trace_c3.txt 2>&1; echo "trace exit $?"
if [ -f paper_2111_05188_b200/libpod_gtime.so ]; then
  for c in C3 C2; do POD_LIB_PATH=$PWD/paper_2111_05188_b200/libpod_gtime.so timeout 200 python tools/fused_probe.py $c; done \
      > $OUT/fused_phases.txt 2>&1; echo "phases exit $?"
fi
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --profile-stride 0 --tdata 100000"
# headline path (the fused rollout kernel at C3) and the separate actor / env-step launches (POD_FUSED=0: the
# path C5 runs), both at the bench's T = 256
$CMD > $OUT/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --cache-control none --csv --log-file $OUT/launches_c3.csv $CMD > $OUT/ncu_list.log 2>&1; echo "list exit $?"
POD_FUSED=0 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --cache-control none --csv --log-file $OUT/launches_c3_sep.csv $CMD > $OUT/ncu_list_sep.log 2>&1; echo "list sep exit $?"
ncu --set full --clock-control none --import-source on -k regex:rollout_fused -s 2 -c 1 -o $OUT/prof_rollout_fused \
    $CMD > $OUT/ncu_rollout_fused.log 2>&1; echo "ncu rollout_fused exit $?"
for K in actor_forward env_step gae; do
  SKIP=20; [ "$K" = gae ] && SKIP=3
  POD_FUSED=0 ncu --set full --clock-control none --import-source on -k regex:$K -s $SKIP -c 1 -o $OUT/prof_$K $CMD \
      > $OUT/ncu_$K.log 2>&1
  echo "ncu $K exit $?"
done
