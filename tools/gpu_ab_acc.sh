# A/B of the deferred scalar reduction of k_bwd_mma (build_variant libraries acc / acc2), run under gpurun.
mkdir -p gpurun_out/ab2
O=gpurun_out/ab2
P=$PWD/paper_2404_02844_b200
for rep in 1 2; do
for v in base acc acc2; do
  L=$P/libqdt_$v.so; [ $v = base ] && L=$P/libqdt.so
  for c in megascale paper_tmd; do
    QDT_LIB=$L timeout 600 python tools/ab_config.py $c 64,200 $v >> $O/ab_$c.jsonl 2>> $O/ab.err
  done
done
done
for v in base acc2; do
  L=$P/libqdt_$v.so; [ $v = base ] && L=$P/libqdt.so
  QDT_LIB=$L AB_ACCEL=1 timeout 600 python tools/ab_config.py megascale 64,200 fista_$v >> $O/ab_megascale.jsonl 2>> $O/ab.err
done
for v in acc2 acc; do
  QDT_LIB=$P/libqdt_$v.so timeout 1500 python -m pytest tests -m gpu -q -x -p no:warnings --deselect tests/test_gpu_round2.py::test_large_200_iterations -k "not stress_shaped and not BB_LS" > $O/pytest_$v.log 2>&1
done
