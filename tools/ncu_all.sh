#!/bin/bash
# ncu evidence for every bench case (run on the GPU box through gpurun, one ncu family per call):
#   launch lists (gpu__time_duration.sum) and one --set full capture of the dominant kernel.
# usage: tools/ncu_all.sh <tag>     -> gpurun_out/ncu_<tag>_*.csv / *.ncu-rep
tag=${1:-r02}
B="--steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
cases=("3::level:translate" "0::p8:translate" "1:m2m:m2m:translate" "1:l2l:l2l:translate" "2::p6:translate" "4:24to12:24to12:translate" "4:12to24:12to24:translate" "4:p30:p30:translate" "4:p16:p16:translate")
for c in "${cases[@]}"; do
  IFS=: read cfg cs name pat <<< "$c"
  args="--config $cfg"; [ -n "$cs" ] && args="$args --case $cs"
  python bench.py $B $args > gpurun_out/plain_$name.log 2>&1 || { echo "plain run failed: $c"; continue; }
  ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/ncu_launches_${tag}_cfg${cfg}_$name.csv python bench.py $B $args > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on -k regex:$pat -s 3 -c 1 -f -o gpurun_out/ncu_full_${tag}_cfg${cfg}_$name python bench.py $B $args > /dev/null 2>&1
done
# gpurun brings back at most 64 MiB: keep the raw-page CSVs of all captures, the reports of
# the level and of configs[0] only
for f in gpurun_out/ncu_full_${tag}_*.ncu-rep; do
  ncu -i $f --page raw --csv > ${f%.ncu-rep}.csv 2>/dev/null
  case $f in *cfg3_level*|*cfg0_p8*) ;; *) rm -f $f ;; esac
done
ls -la gpurun_out/ | grep ncu_ | tail -30
