# A/B of the integer-key bounds in the N-split FISTA step kernel (build_variant library ikp), run under gpurun.
mkdir -p gpurun_out/ab4
O=gpurun_out/ab4
P=$PWD/paper_2404_02844_b200
for rep in 1 2; do
for v in base ikp; do
  L=$P/libqdt_$v.so; [ $v = base ] && L=$P/libqdt.so
  QDT_LIB=$L AB_ACCEL=1 timeout 600 python tools/ab_config.py megascale 64,200 fista_$v >> $O/ab_megascale_fista.jsonl 2>> $O/ab.err
done
done
QDT_LIB=$P/libqdt_ikp.so timeout 1500 python -m pytest tests -m gpu -q -x -p no:warnings -k "fista or resume or virtual or tiny or medium_solve or early_stop" > $O/pytest_ikp.log 2>&1
