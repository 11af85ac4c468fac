# one GPU, round-2 final lines: default bench (config 3) with e2e + cpu_baseline, reference arm, every config,
# whole-workload runs, ncu launch list + full capture of config 3 and config 2, SASS summary
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py --steps 2000 --warmup 20 > gpurun_out/fin_c3_g1.json 2> gpurun_out/fin_c3_g1.err; echo c3 rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err; echo ref rc=$?
for C in 2 5a 5b 5c 5d; do
timeout 900 python bench.py --config $C --steps $([ $C = 2 ] && echo 5000 || echo 200) --warmup 20 --no-cpu-baseline > gpurun_out/fin_c${C}_g1.json 2> gpurun_out/fin_c${C}_g1.err; echo c$C rc=$?
done
timeout 900 python bench.py --config 1 --steps 200 --warmup 5 > gpurun_out/fin_c1_g1.json 2> gpurun_out/fin_c1_g1.err; echo c1 rc=$?
timeout 900 python bench.py --config 4 --steps 3 --warmup 1 > gpurun_out/fin_c4_g1.json 2> gpurun_out/fin_c4_g1.err; echo c4 rc=$?
timeout 900 python bench.py --config 2 --workload > gpurun_out/fin_wl2_g1.json 2> gpurun_out/fin_wl2_g1.err; echo wl2 rc=$?
timeout 900 python bench.py --config 3 --workload > gpurun_out/fin_wl3_g1.json 2> gpurun_out/fin_wl3_g1.err; echo wl3 rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin_launches_c3.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/fin_launches.log 2>&1; echo launches rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"asp_replay|bsp_update" -s 10 -c 2 -o gpurun_out/fin_ncu_c3 -f python bench.py --config 3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/fin_ncu_c3.log 2>&1; echo ncu3 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"asp_replay|bsp_update" -s 40 -c 2 -o gpurun_out/fin_ncu_c2 -f python bench.py --config 2 --steps 40 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/fin_ncu_c2.log 2>&1; echo ncu2 rc=$?
timeout 900 ncu --set full --clock-control none -k regex:"asp_replay|bsp_update" -s 4 -c 2 -o gpurun_out/fin_ncu_c5a -f python bench.py --config 5a --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/fin_ncu_c5a.log 2>&1; echo ncu5a rc=$?
