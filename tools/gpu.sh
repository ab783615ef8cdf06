#!/usr/bin/env bash
# One entry point for the GPU-box steps (run through gpurun from the repo root):
#   bash tools/gpu.sh <step> [<step> ...]
# steps:
#   build      compile the CUDA library + oracle (__graft_entry__.build)
#   smoke      __graft_entry__.smoke()
#   test       pytest -m gpu (without the slow 1B tests)
#   testall    pytest -m gpu (everything, incl. the 1B config-4 pin)
#   sanitize   compute-sanitizer memcheck / racecheck / synccheck / initcheck
#              of tools/sanitize.py  -> gpurun_out/sanitize_<tool>.log
#   bench      bench.py headline (100M float3 RR) + widest config 5 + reference arm
#   launches   ncu launch lists (time + DRAM bytes per launch) of one 100M RR and
#              one 100M clustered widest build -> gpurun_out/launches_*.{csv,txt}
#   full       ncu --set full captures of the partition / in-CTA / filter kernels
#   robust     tools/robust_time.py + tools/quick_time.py
#   degen      ncu launch lists of adversarial 10M builds (identical, huge range, constant axis, ties)
#   evidence   the round's committed evidence (launch lists, ncu captures, robustness and config timings)
#   knobs      tools/knobs.py: per-kernel-class times under env variants ($KNOBS)
#   big        tools/big_build.py (1B clustered, sharded decomposition on one GPU)
# Env: TEST_ARGS (extra pytest args), KSEL (ncu kernel regex for `full`, default all three)
set -u
mkdir -p gpurun_out
step_build() { python __graft_entry__.py build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }; }
step_smoke() { timeout 300 python __graft_entry__.py 2>&1 | tail -2; }
step_test() { timeout 2400 python -m pytest tests/ -q -m "gpu and not slow" ${TEST_ARGS:-} 2>&1 | tail -25; }
step_testall() { timeout 3000 python -m pytest tests/ -q -m gpu ${TEST_ARGS:-} 2>&1 | tail -25; }
step_sanitize() {
  for tool in memcheck racecheck synccheck initcheck; do
    LBKD_GRAPH=0 timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize.py 200000 \
      > gpurun_out/sanitize_$tool.log 2>&1
    echo "== $tool rc=$?"; tail -4 gpurun_out/sanitize_$tool.log
  done
}
step_bench() {
  timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log > gpurun_out/bench.json; cut -c1-400 gpurun_out/bench.json
  timeout 900 python bench.py --steps 10 --warmup 3 --mode widest --dist clustered --no-cpu-baseline > gpurun_out/bench_widest.log 2>&1; tail -1 gpurun_out/bench_widest.log > gpurun_out/bench_widest.json; cut -c1-400 gpurun_out/bench_widest.json
  timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log > gpurun_out/bench_ref.json; cut -c1-400 gpurun_out/bench_ref.json
}
step_launches() {
  L=$(python tools/one_build.py 100000000 3 rr uniform 1 | awk '/launches per build/{print $4}')
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s $L -c $L --csv --log-file gpurun_out/launches_100m.csv python tools/one_build.py 100000000 3 rr uniform 2 > gpurun_out/prof1.log 2>&1
  python tools/launches.py gpurun_out/launches_100m.csv > gpurun_out/launches_100m.txt
  python tools/ncu_traffic.py gpurun_out/launches_100m.csv gpurun_out/ncu_traffic.json > /dev/null
  L=$(python tools/one_build.py 100000000 3 widest clustered 1 | awk '/launches per build/{print $4}')
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s $L -c $L --csv --log-file gpurun_out/launches_widest.csv python tools/one_build.py 100000000 3 widest clustered 2 > gpurun_out/profw1.log 2>&1
  python tools/launches.py gpurun_out/launches_widest.csv > gpurun_out/launches_widest.txt
  python tools/ncu_traffic.py gpurun_out/launches_widest.csv gpurun_out/ncu_traffic_widest.json > /dev/null
  cat gpurun_out/launches_100m.txt gpurun_out/launches_widest.txt | head -80
}
step_full() {
  for ks in ${KSEL:-sel_part subtree sel_filter}; do
    skip=0; [ "$ks" = sel_part ] && skip=4; [ "$ks" = sel_filter ] && skip=6
    ncu --set full --clock-control none --import-source on -k regex:$ks -s $skip -c 1 -o gpurun_out/full_$ks python tools/one_build.py 100000000 3 rr uniform 1 > gpurun_out/full_$ks.log 2>&1
    python tools/ncu_lines.py gpurun_out/full_$ks.ncu-rep 60 > gpurun_out/full_${ks}_lines.txt 2>&1
    python tools/ncu_issue.py gpurun_out/full_$ks.ncu-rep gpurun_out/ncu_issue_$ks.json > /dev/null 2>&1
    ncu -i gpurun_out/full_$ks.ncu-rep --page details --csv > gpurun_out/full_${ks}_details.csv 2>/dev/null
  done
}
step_robust() {
  timeout 600 python tools/robust_time.py > gpurun_out/robust_time.txt 2>&1; cat gpurun_out/robust_time.txt
  timeout 300 python tools/quick_time.py > gpurun_out/quick_time.txt 2>&1; cat gpurun_out/quick_time.txt
}
step_degen() {  # ncu launch lists of adversarial 10M builds (where the time goes)
  for kind in identical huge constaxis ties; do
    for mode in rr widest; do
      L=$(python tools/one_build.py 10000000 3 $mode $kind 1 | awk '/launches per build/{print $4}')
      ncu --metrics gpu__time_duration.sum --clock-control none -s $L -c $L --csv --log-file gpurun_out/degen_${kind}_$mode.csv python tools/one_build.py 10000000 3 $mode $kind 2 > /dev/null 2>&1
      echo "== $kind $mode"; python tools/launches.py gpurun_out/degen_${kind}_$mode.csv | head -14
    done
  done
}
step_knobs() {  # per-class times of 100M builds under tuning switches (KNOBS overrides the list)
  python tools/knobs.py 100000000 3 rr uniform -- ${KNOBS:-"" LBKD_SUBTREE_BITS=11 LBKD_SUBTREE=sel}
  python tools/knobs.py 100000000 3 widest clustered -- ${KNOBS:-"" LBKD_SUBTREE_BITS=11 LBKD_SUBTREE=sel}
}
step_evidence() {  # the round's committed evidence -> gpurun_out/r02_* (copied to profiles/ by hand)
  R=gpurun_out/r02
  L=$(python tools/one_build.py 100000000 3 rr uniform 1 | awk '/launches per build/{print $4}')
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s $L -c $L --csv --log-file ${R}_launches_100m_float3.csv python tools/one_build.py 100000000 3 rr uniform 2 > /dev/null 2>&1
  python tools/launches.py ${R}_launches_100m_float3.csv > ${R}_launches_100m_float3.txt
  python tools/ncu_traffic.py ${R}_launches_100m_float3.csv ${R}_ncu_traffic.json > /dev/null
  L=$(python tools/one_build.py 100000000 3 widest clustered 1 | awk '/launches per build/{print $4}')
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s $L -c $L --csv --log-file ${R}_launches_100m_clustered_widest.csv python tools/one_build.py 100000000 3 widest clustered 2 > /dev/null 2>&1
  python tools/launches.py ${R}_launches_100m_clustered_widest.csv > ${R}_launches_100m_clustered_widest.txt
  python tools/ncu_traffic.py ${R}_launches_100m_clustered_widest.csv ${R}_ncu_traffic_widest.json > /dev/null
  # round robin: the pair kernels (4th launch = levels 6/7), the single-level
  # partition / filter (last global level), the in-CTA kernel
  for spec in sel_part_pair:3 sel_filter_pair:3 sel_child_hist:3 sel_part_bulk:0 sel_filter_kernel:4 subtree:0; do
    ks=${spec%%:*}; skip=${spec##*:}
    ncu --set full --clock-control none --import-source on -k regex:$ks -s $skip -c 1 -o ${R}_full_$ks python tools/one_build.py 100000000 3 rr uniform 1 > /dev/null 2>&1
    python tools/ncu_summary.py ${R}_full_$ks.ncu-rep > ${R}_ncu_full_$ks.txt 2>&1
    python tools/ncu_lines.py ${R}_full_$ks.ncu-rep 60 > ${R}_ncu_lines_$ks.txt 2>&1
  done
  # widest: its single-level partition (5th launch)
  ncu --set full --clock-control none --import-source on -k regex:sel_part_bulk -s 4 -c 1 -o ${R}_full_part_widest python tools/one_build.py 100000000 3 widest clustered 1 > /dev/null 2>&1
  python tools/ncu_summary.py ${R}_full_part_widest.ncu-rep > ${R}_ncu_full_part_widest.txt 2>&1
  python tools/ncu_issue.py ${R}_full_subtree.ncu-rep ${R}_ncu_issue_subtree.json > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on -k regex:subtree -c 1 -o ${R}_full_subsel_widest python tools/one_build.py 100000000 3 widest clustered 1 > /dev/null 2>&1
  python tools/ncu_summary.py ${R}_full_subsel_widest.ncu-rep > ${R}_ncu_full_subsel_widest.txt 2>&1
  python tools/ncu_issue.py ${R}_full_subsel_widest.ncu-rep ${R}_ncu_issue_subtree_widest.json > /dev/null 2>&1
  rm -f ${R}_full_*.ncu-rep
  { for kind in uniform clustered identical huge constaxis ties sorted; do
      KNOBS_TIMEOUT=120 python tools/knobs.py 10000000 3 rr $kind -- ""; KNOBS_TIMEOUT=120 python tools/knobs.py 10000000 3 widest $kind -- ""
    done; KNOBS_TIMEOUT=120 python tools/knobs.py 100000000 3 rr ties -- ""; } > ${R}_robust_knobs.txt 2>&1
  { KNOBS_TIMEOUT=300 python tools/knobs.py 100000000 3 rr uniform -- "" LBKD_PAIR=0 LBKD_ALGO=sort LBKD_SELECT_CLUSTER=0
    KNOBS_TIMEOUT=120 python tools/knobs.py 100000000 2 rr uniform -- ""
    KNOBS_TIMEOUT=120 python tools/knobs.py 10000000 4 rr uniform -- ""
    KNOBS_TIMEOUT=120 python tools/knobs.py 1000000 3 rr uniform -- ""
    KNOBS_TIMEOUT=120 python tools/knobs.py 100000000 3 widest clustered -- ""
    KNOBS_TIMEOUT=120 python tools/knobs.py 100000000 3 rr clustered -- "" LBKD_PAIR=0
    KNOBS_TIMEOUT=300 python tools/knobs.py 100000000 3 rr uniform64 -- ""
    KNOBS_TIMEOUT=300 python tools/knobs.py 10000000 4 rr uniform64 -- ""; } > ${R}_configs_knobs.txt 2>&1
  cat ${R}_launches_100m_float3.txt | head -20
}
step_big() { timeout 900 python tools/big_build.py 1000000000 clustered 3 > gpurun_out/big_1b.log 2>&1; tail -1 gpurun_out/big_1b.log | cut -c1-600; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv,noheader
for s in "$@"; do echo "=== $s"; step_$s; done
