# ncu full captures of the secondary kernels (batched jump, bank Langevin, persistence)
mkdir -p gpurun_out
for c in jump bank text; do timeout 300 python tools/profile_case.py $c > gpurun_out/plain_$c.log 2>&1; echo plain_$c=$?; done
timeout 900 ncu --set full --clock-control none -k regex:apply2 -s 2 -c 1 -o gpurun_out/full_apply2 python tools/profile_case.py jump > gpurun_out/ncu_f_jump.log 2>&1; echo apply2=$?
timeout 900 ncu --set full --clock-control none -k regex:langevin_bank -s 2 -c 1 -o gpurun_out/full_bank python tools/profile_case.py bank > gpurun_out/ncu_f_bank.log 2>&1; echo bank=$?
timeout 900 ncu --set full --clock-control none -k regex:"to_text_kernel|from_text_warp|text_len" -s 3 -c 3 -o gpurun_out/full_text python tools/profile_case.py text > gpurun_out/ncu_f_text.log 2>&1; echo text=$?
