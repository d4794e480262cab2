mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/f_t.log 2>&1; echo "pytest rc $?" >> gpurun_out/f_t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/f_smoke.log
timeout 300 python bench.py > gpurun_out/f_b.json 2>gpurun_out/f_b.err
AFS_STAGE_STREAMS=1 timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/f_b_1s.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/f_ncu_l.log 2>&1
timeout 600 ncu -f --set full --import-source on --clock-control none -k regex:'k_(gather|spread)_tc' -c 2 -o /tmp/g3 python tools/profile_c3.py --windows 0,3 --applies 1 > gpurun_out/f_ncu_g.log 2>&1
ncu -i /tmp/g3.ncu-rep --page raw --csv > gpurun_out/f_g_raw.csv 2>&1
ncu -i /tmp/g3.ncu-rep --page source --csv > gpurun_out/f_g_src.csv 2>&1
