# Round 2 (session 4 (end)) final evidence at HEAD: whole GPU suite, smoke, both bench arms,
# launch lists and one ncu --set full capture per hot kernel. Outputs under gpurun_out/final5/.
mkdir -p gpurun_out/final5
O=gpurun_out/final5
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt
nproc > $O/nproc.txt
timeout 1500 python -m pytest tests -m gpu -q -rs > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 $O/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > $O/bench.log 2>&1; echo bench=$?
timeout 1200 python bench.py --impl reference > $O/bench_ref.log 2>&1; echo bench_ref=$?
timeout 300 python tools/time_k4.py > $O/time_k4.log 2>&1; echo time_k4=$?
timeout 300 python tools/time_c4.py > $O/time_c4.log 2>&1; echo time_c4=$?
for c in c1 c2 c3 c4 c5 lang bank jump text; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_$c.csv python tools/profile_case.py $c > /dev/null 2>&1; echo launches_$c=$?
done
full() { timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s ${4:-2} -c 1 -o $O/full_$1 python tools/profile_case.py $3 $5 > /dev/null 2>&1; echo full_$1=$?; }
full gen_store gen_store c2
full bulk_tc bulk_tc c3 3
full consume consume c4 0 "--warmup 0 --c4-streams 1048576"
full gaussian gaussian_kernel c5
full langevin langevin_kernel lang
full bank langevin_bank bank
full apply_tc apply_tc jump
full to_text to_text_kernel text
full from_text from_text_warp_kernel text
timeout 300 python tools/time_text.py > $O/time_text.log 2>&1; echo time_text=$?
timeout 300 python tools/time_c1.py > $O/time_c1.log 2>&1; echo time_c1=$?
