# Quick ncu metric comparison of one kernel between the in-tree library and variants.
# usage: bash tools/gpu_ncu_ab.sh <kernel-regex> "<bench args>" lib1 lib2 ...
O=gpurun_out/ncu_ab
mkdir -p $O
k=$1; shift; args=$1; shift
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,sm__warps_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed,smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio
for lib in "" "$@"; do
  n=$(basename "${lib:-default}" .so)
  DIVUQ_LIB_PATH=$lib ncu --metrics $M --clock-control none -k regex:$k -s 3 -c 1 --csv --log-file $O/$n.csv python bench.py $args --no-e2e --no-cpu --no-fp64 > /dev/null 2> $O/$n.err
  python - "$O/$n.csv" "$n" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and not r[0].startswith("==")]
hdr = rows[0]; mi = hdr.index("Metric Name"); vi = hdr.index("Metric Value")
print("==", sys.argv[2])
for r in rows[1:]:
    print("  %-90s %s" % (r[mi], r[vi]))
PY
done
