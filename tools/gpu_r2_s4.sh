# Session 4: GPU suite, smoke and both bench arms at HEAD + K7 text launch list and ncu captures.
O=gpurun_out/s4
mkdir -p $O
timeout 300 python tools/time_text.py > $O/time_text.log 2>&1; echo time_text=$?; cat $O/time_text.log
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_text.csv python tools/time_text.py --reps 1 > $O/ncu_text_l.log 2>&1; echo ncu_l=$?
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on \
  -k regex:"to_text_kernel|from_text_warp_kernel" -c 2 -o $O/text_full -f \
  python tools/time_text.py --reps 1 > $O/ncu_text_f.log 2>&1; echo ncu_f=$?
timeout 1500 python -m pytest tests -m gpu -q -rs > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 $O/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > $O/bench.log 2>&1; echo bench=$?
timeout 1200 python bench.py --impl reference > $O/bench_ref.log 2>&1; echo bench_ref=$?
