for i in 1 2; do
for L in paper_2602_15922_b200/libdz_old.so paper_2602_15922_b200/libdz.so; do
echo -n "$L: "; DZ_LIB_PATH=$PWD/$L timeout 200 python bench.py --no-cpu-baseline --e2e-steps 0 --steps 100 > /tmp/b.json 2>/dev/null; python tools/bench_brief.py /tmp/b.json
done; done
