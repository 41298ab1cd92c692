# Round 2 profiles: launch lists per config (cold, serialised) and one
# ncu --set full capture per hot kernel. Outputs under gpurun_out/prof/.
mkdir -p gpurun_out/prof
for c in c2 c3 c4 c5 lang bank jump; do
  timeout 300 python tools/profile_case.py $c > gpurun_out/prof/plain_$c.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/prof/launches_$c.csv python tools/profile_case.py $c > gpurun_out/prof/ncu_l_$c.log 2>&1; echo launches_$c=$?
done
full() { timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s ${4:-2} -c 1 -o gpurun_out/prof/full_$1 python tools/profile_case.py $3 > gpurun_out/prof/ncu_f_$1.log 2>&1; echo full_$1=$?; }
full gen_store gen_store c2
full bulk_tc bulk_tc c3
full consume consume c4
full gaussian gaussian_kernel c5
full langevin langevin_kernel lang
full bank langevin_bank bank
full apply2 apply2 jump
