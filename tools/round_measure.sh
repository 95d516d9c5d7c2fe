#!/bin/bash
# Round-end measurement set (one B200): bench lines, launch lists, one ncu --set full capture of
# the dominant kernel.  Every ncu command runs only after the same command exited 0 without ncu.
set -u
O=gpurun_out/final
mkdir -p $O
python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo "bench c3 rc=$?"
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
for c in c1 c2 c4; do python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c rc=$?"; done
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"stats|decide|resample" -c 24 --csv \
      --log-file $O/launches_c3.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "launches c3 rc=$?"
python bench.py --config c4 --steps 3 --warmup 3 --no-e2e > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"stats|tree" -c 12 --csv \
      --log-file $O/launches_c4.csv python bench.py --config c4 --steps 3 --warmup 3 > /dev/null 2>&1; echo "launches c4 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:stats_kernel -s 4 -c 1 -o /tmp/stats_c3 \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu -i /tmp/stats_c3.ncu-rep --page details --csv > $O/stats_c3_details.csv 2>&1
ncu -i /tmp/stats_c3.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread > $O/stats_c3_raw.csv 2>&1
ncu --set full --clock-control none -k regex:resample_kernel -s 4 -c 1 -o /tmp/res_c3 \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu resample rc=$?"
ncu -i /tmp/res_c3.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > $O/resample_c3_raw.csv 2>&1
ls -la $O
