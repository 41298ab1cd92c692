# batched jump_state: parity tests + 2^20 jumps at J = 2^120
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ranmars.py tests/test_facade.py -q -x -k "jump or make_streams or config3 or ranmars or facade" > gpurun_out/ap_pt.log 2>&1; echo pt=$?; tail -2 gpurun_out/ap_pt.log
timeout 300 python - <<'PY'
import torch, paper_2512_00093_b200 as rb
n=1<<20
st=rb.make_streams(12345,2**40,n); out=torch.empty_like(st)
for _ in range(3): rb.jump_dev(st,2**120,out=out)
torch.cuda.synchronize(); ts=[]
for r in range(5):
    a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    a.record(); rb.jump_dev(st,2**120,out=out); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
print("batched jump ms", ["%.3f"%t for t in ts], int(out.sum()))
PY
