# Round 2: integer-pipe peaks (config-3 / config-4 roofline denominators) and a
# whole-config ncu capture of K2 (config 4 at 2^20 streams = 18.4 waves).
mkdir -p gpurun_out
make -s lib micro >/dev/null
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_throttle_reasons.active --format=csv -lms 200 > gpurun_out/int_clocks.csv &
SMI=$!
timeout 300 tools/micro/intpipes > gpurun_out/intpipes_maxclk.txt 2>&1; echo intpipes=$?
kill $SMI
CLK=$(awk -F, 'NR>1 {gsub(/ MHz/,"",$1); print $1+0}' gpurun_out/int_clocks.csv | sort -n | awk '{a[NR]=$1} END {print a[int(NR*0.75)]}')
timeout 300 tools/micro/intpipes $CLK > gpurun_out/intpipes.txt 2>&1; echo intpipes_clk=$CLK
timeout 600 python tools/profile_case.py c4 --c4-streams 1048576 --warmup 1 > gpurun_out/plain_c4full.log 2>&1; echo plain_c4=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:consume -s 1 -c 1 -o gpurun_out/full_consume_c4full python tools/profile_case.py c4 --c4-streams 1048576 --warmup 1 > gpurun_out/ncu_f_c4full.log 2>&1; echo full_c4=$?
