# ncu --set full of the LCP kernels at HEAD -> summaries, SASS mix, pipe utilisation
O=gpurun_out
for pair in "lcp2d_tma:lcp" "lcp2d_fused:lcpfused"; do
  k=${pair%%:*}; w=${pair##*:}
  ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o $O/prof_$k python bench.py --workload $w --steps 3 --no-e2e --no-cpu > $O/ncu_$k.log 2>&1
  python tools/ncu_summary.py $O/prof_$k.ncu-rep > $O/${k}_summary.txt
  ncu -i $O/prof_$k.ncu-rep --page source --csv --print-source sass > $O/src_$k.csv 2>/dev/null
  python tools/sass_mix_csv.py $O/src_$k.csv > $O/${k}_sassmix.txt; rm -f $O/src_$k.csv
  ncu -i $O/prof_$k.ncu-rep --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
for k,x in zip(h,v):
  if any(s in k for s in ('pipe_fp64','pipe_fma','pipe_alu','lsu_wavefronts','issue_active','dram__throughput')) and 'pct' in k and '.max' not in k and '.min' not in k: print(k,x)
" > $O/${k}_pipes.txt
  rm -f $O/prof_$k.ncu-rep
done
