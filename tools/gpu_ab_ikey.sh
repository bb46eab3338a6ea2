# A/B of the integer-key row epilogue variants (build_variant libraries) + one ncu capture of
# k_bwd_mma with the warp-stall breakdown (run under gpurun).
mkdir -p gpurun_out/ab
O=gpurun_out/ab
P=$PWD/paper_2404_02844_b200
for rep in 1 2; do
for v in base ikey iclamp ikc; do
  L=$P/libqdt_$v.so; [ $v = base ] && L=$P/libqdt.so
  for c in megascale paper_tmd; do
    QDT_LIB=$L timeout 600 python tools/ab_config.py $c 64,200 $v >> $O/ab_$c.jsonl 2>> $O/ab.err
  done
done
done
for v in base ikc; do
  L=$P/libqdt_$v.so; [ $v = base ] && L=$P/libqdt.so
  QDT_LIB=$L AB_ACCEL=1 timeout 600 python tools/ab_config.py megascale 64,200 fista_$v >> $O/ab_megascale.jsonl 2>> $O/ab.err
  QDT_LIB=$L timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:warnings -k "projection or one_step or medium or tiny or shape_edges or long_axis" > $O/pytest_$v.log 2>&1
done
CMD="python bench.py --config megascale --steps 4 --warmup 3 --no-cpu --no-e2e --no-ttt"
for v in base ikc; do
  L=$P/libqdt_$v.so; [ $v = base ] && L=$P/libqdt.so
  QDT_LIB=$L timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:k_bwd_mma -s 4 -c 1 -o /tmp/prof_$v $CMD > $O/ncu_$v.log 2>&1
  ncu -i /tmp/prof_$v.ncu-rep --page raw --csv > $O/raw_$v.csv 2>&1
  ncu -i /tmp/prof_$v.ncu-rep --page details --csv > $O/details_$v.csv 2>&1
  ncu -i /tmp/prof_$v.ncu-rep --page source --csv --print-source cuda,sass > /tmp/src_$v.csv 2>&1
  python tools/ncu_src_summary.py /tmp/src_$v.csv 40 > $O/src_$v.txt 2>&1
  python tools/ncu_details_summary.py $O/details_$v.csv > $O/summary_$v.txt 2>&1
done
