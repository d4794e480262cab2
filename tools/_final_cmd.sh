mkdir -p gpurun_out
timeout 600 ncu -f --set full --import-source on --clock-control none -k regex:'k_(gather|spread)_tc' -c 2 -o /tmp/g2 python tools/profile_c3.py --windows 0,3 --applies 1 > gpurun_out/f_ncu_g.log 2>&1
ncu -i /tmp/g2.ncu-rep --page raw --csv > gpurun_out/f_g_raw.csv 2>&1
python tools/ncu_summary.py /tmp/g2.ncu-rep > gpurun_out/f_g_summary.txt 2>&1
