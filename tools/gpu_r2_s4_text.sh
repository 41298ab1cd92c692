# Session 4: K7 one-pass to_text + SWAR from_text: parity, timing, sanitizers, launch list, ncu.
O=gpurun_out/s4t
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_text.py tests/test_cli.py tests/test_gpu_parity.py -q -x -k "text or cli or invalid or empty" > $O/pt.log 2>&1; echo pt=$?; tail -3 $O/pt.log
timeout 300 python tools/time_text.py > $O/time_text.log 2>&1; echo time_text=$?; cat $O/time_text.log
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck python tools/sanitize_case.py > $O/memcheck.log 2>&1; echo memcheck=$?; tail -3 $O/memcheck.log
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool racecheck python tools/sanitize_case.py > $O/racecheck.log 2>&1; echo racecheck=$?; tail -3 $O/racecheck.log
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_text.csv python tools/time_text.py --reps 1 > $O/ncu_text_l.log 2>&1; echo ncu_l=$?
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on \
  -k regex:"to_text_kernel|from_text_warp_kernel" -c 2 -o $O/text_full -f \
  python tools/time_text.py --reps 1 > $O/ncu_text_f.log 2>&1; echo ncu_f=$?
