#!/bin/bash
# Round-2 session-5 captures (run under gpurun, 1 GPU): each command runs once
# plainly (must exit 0), then under ncu --set full.  Reports stay in /tmp on
# the box; the text summaries (and reports under 12 MiB) come back.
OUT=${OUT:-gpurun_out}
T=/tmp/ncu_s5
mkdir -p $OUT $T
NCU="ncu --set full --clock-control none --import-source on"
cap() {  # name kernel-regex skip count cmd...
  local name=$1 rx=$2 skip=$3 cnt=$4; shift 4
  "$@" > $OUT/plain_$name.log 2>&1 || { echo "$name: plain run failed"; return; }
  $NCU -k "regex:$rx" -s $skip -c $cnt -o $T/$name -f "$@" > $OUT/ncu_$name.log 2>&1
  ncu -i $T/$name.ncu-rep --page raw --csv > $OUT/$name.raw.csv 2>/dev/null
  python tools/ncu_hot.py $T/$name.ncu-rep 40 > $OUT/$name.hot.txt 2>&1
  python tools/ncu_lines.py $T/$name.ncu-rep 60 > $OUT/$name.lines.txt 2>&1
  local sz=$(stat -c %s $T/$name.ncu-rep)
  [ "$sz" -lt 12000000 ] && cp $T/$name.ncu-rep $OUT/
}
for what in "$@"; do
  case $what in
    seg) cap seg_s5 seg_kernel 1 1 python tools/workloads.py --which cfg4 --reps 1 ;;
    pkfew) cap pkfew_s5 pksort_kernel 1 1 python tools/pk_one.py 256 few16 merge ;;
    pkuni) cap pkuni_s5 pksort_kernel 1 1 python tools/pk_one.py 256 uniform merge ;;
    pkrss) cap pkrss_s5 pksort_kernel 1 1 python tools/pk_one.py 256 uniform rss ;;
    pkrss32) cap pkrss32_s5 pksort_kernel 1 1 python tools/pk_one.py 32 uniform rss ;;
    pkrss64) cap pkrss64_s5 pksort_kernel 1 1 python tools/pk_one.py 64 uniform rss ;;
    pkmrg32) cap pkmrg32_s5 pksort_kernel 1 1 python tools/pk_one.py 32 uniform merge ;;
    pkmrg64) cap pkmrg64_s5 pksort_kernel 1 1 python tools/pk_one.py 64 uniform merge ;;
    pkref) cap pkref_s5 pksort_kernel 1 1 python tools/ref_probe.py --ns 256 --reps 1 ;;
    launches)
      python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --workloads none > $OUT/plain_launch.log 2>&1 && \
      ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
        python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --workloads none > $OUT/ncu_launch.log 2>&1 ;;
    net7) cap net7_s5 "net_|nettma|netbulk" 4 4 python bench.py --ns 7 --steps 1 --warmup 1 --no-e2e --no-cpu --workloads none ;;
    net10) cap net10_s5 "net_|nettma|netbulk" 4 4 python bench.py --ns 10 --steps 1 --warmup 1 --no-e2e --no-cpu --workloads none ;;
  esac
done
echo done
