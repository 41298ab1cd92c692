mkdir -p gpurun_out
for n in 1 129 100000; do timeout 120 python tools/time_c3.py --n $n --reps 2 --compare 2>&1 | tail -1; done
timeout 300 python tools/time_c3.py --compare > gpurun_out/tc_full4.log 2>&1; echo full=$?; tail -3 gpurun_out/tc_full4.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bulk_tc -s 3 -c 1 -o gpurun_out/bulk_tc3 python tools/time_c3.py --reps 1 > gpurun_out/tcncu.log 2>&1; echo ncu=$?
