# Round 2 final evidence: whole GPU suite, smoke, both bench arms, launch lists
# and one ncu --set full capture per hot kernel. Outputs under gpurun_out/final/.
mkdir -p gpurun_out/final
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/final/gpu.txt
nproc > gpurun_out/final/nproc.txt
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/final/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/final/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/final/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/final/bench.log 2>&1; echo bench=$?
timeout 1200 python bench.py --impl reference > gpurun_out/final/bench_ref.log 2>&1; echo bench_ref=$?
for c in c2 c3 c4 c5 lang bank jump; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/final/launches_$c.csv python tools/profile_case.py $c > /dev/null 2>&1; echo launches_$c=$?
done
full() { timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s ${4:-2} -c 1 -o gpurun_out/final/full_$1 python tools/profile_case.py $3 > /dev/null 2>&1; echo full_$1=$?; }
full gen_store gen_store c2
full bulk_tc bulk_tc c3 3
full consume consume c4
full gaussian gaussian_kernel c5
full langevin langevin_kernel lang
full bank langevin_bank bank
full apply_tc apply_tc jump
