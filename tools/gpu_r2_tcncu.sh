mkdir -p gpurun_out
timeout 300 python tools/time_c3.py --compare > gpurun_out/tc_full2.log 2>&1; echo full=$?; tail -3 gpurun_out/tc_full2.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bulk_tc -s 3 -c 1 -o gpurun_out/bulk_tc python tools/time_c3.py --reps 1 > gpurun_out/tcncu.log 2>&1; echo ncu=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_tc.csv python tools/profile_case.py c3 > gpurun_out/tcl.log 2>&1; echo launches=$?
