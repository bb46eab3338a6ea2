# A/B of build_variant libraries against the default one (run under gpurun from the repo root).
# Build the variants first, here: python -c "from paper_2404_02844_b200 import build as b; b.build_variant('tag', ['MACRO=1'])"
#   VARIANTS="tag1 tag2"   libqdt_<tag>.so next to libqdt.so ("base" = the default library, always run)
#   CONFIGS="megascale paper_tmd"   qdt_synth configurations     KS="64,200"   iteration counts per call
#   ACCEL=1   also time SQS-FISTA     TESTS="-k ..."   pytest selection run with each variant library
#   NCU=1     one ncu --set full capture of $KERNEL (default k_bwd_mma) per library, with stall summary
O=gpurun_out/ab; mkdir -p $O
P=$PWD/paper_2404_02844_b200
lib() { [ "$1" = base ] && echo $P/libqdt.so || echo $P/libqdt_$1.so; }
for rep in 1 2; do
  for v in base $VARIANTS; do
    for c in ${CONFIGS:-megascale}; do
      QDT_LIB=$(lib $v) timeout 600 python tools/ab_config.py $c ${KS:-64,200} $v >> $O/ab_$c.jsonl 2>> $O/ab.err
      [ -n "$ACCEL" ] && QDT_LIB=$(lib $v) AB_ACCEL=1 timeout 600 python tools/ab_config.py $c ${KS:-64,200} fista_$v >> $O/ab_$c.jsonl 2>> $O/ab.err
    done
  done
done
if [ -n "$TESTS" ]; then
  for v in $VARIANTS; do
    QDT_LIB=$(lib $v) timeout 1800 python -m pytest tests -m gpu -q -x -p no:warnings $TESTS > $O/pytest_$v.log 2>&1
  done
fi
if [ -n "$NCU" ]; then
  CMD="python bench.py --config ${NCU_CFG:-megascale} --steps 4 --warmup 3 --no-cpu --no-e2e --no-ttt"
  for v in base $VARIANTS; do
    QDT_LIB=$(lib $v) timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:${KERNEL:-k_bwd_mma} -s 4 -c 1 -o /tmp/prof_$v $CMD > $O/ncu_$v.log 2>&1
    ncu -i /tmp/prof_$v.ncu-rep --page raw --csv > $O/raw_$v.csv 2>&1
    ncu -i /tmp/prof_$v.ncu-rep --page details --csv > $O/details_$v.csv 2>&1
    ncu -i /tmp/prof_$v.ncu-rep --page source --csv --print-source cuda,sass > /tmp/src_$v.csv 2>&1
    python tools/ncu_src_summary.py /tmp/src_$v.csv 40 > $O/src_$v.txt 2>&1
    python tools/ncu_details_summary.py $O/details_$v.csv > $O/summary_$v.txt 2>&1
    python tools/ncu_stalls.py $O/raw_$v.csv > $O/stalls_$v.txt 2>&1
  done
fi
