# A/B of tuning builds on the bench system (930^3, p = 3): times + digests,
# then DRAM bytes of pass A per build (ncu, 4 launches each)
mkdir -p gpurun_out
PROD=paper_1904_03057_b200/libbspde_b200.so
for round in 1 2; do
  for lib in $PROD "$@"; do
    BSPDE_LIB=$lib timeout 600 python tools/ab_sep.py 930 3 >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
  done
done
for lib in $PROD "$@"; do
  n=$(basename $lib .so)
  BSPDE_LIB=$lib timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:sep_kernel --launch-skip 24 --launch-count 6 --csv \
    --log-file gpurun_out/ncu_$n.csv python tools/ab_sep.py 930 3 > /dev/null 2>> gpurun_out/ab.err
done
cat gpurun_out/ab.jsonl
