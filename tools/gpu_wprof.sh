mkdir -p gpurun_out
for c in stress_cut stress; do
QDT_LIB=paper_2404_02844_b200/libqdt_wprof.so timeout 900 python bench.py --config $c --steps 16 --warmup 3 --no-cpu --no-ttt --no-e2e > gpurun_out/wprof_$c.json 2> gpurun_out/wprof_$c.err
done
