mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "consume or config4" > gpurun_out/c4_pt.log 2>&1; echo pt=$?; tail -2 gpurun_out/c4_pt.log
timeout 300 python - <<'PY'
import torch, paper_2512_00093_b200 as rb
n=1<<20
st=rb.make_streams(42,2**64,n)
s0=st.clone()
rb.consume(st,1<<16); torch.cuda.synchronize()
ts=[]
for r in range(3):
    st.copy_(s0); torch.cuda.synchronize()
    a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    a.record(); sums,h=rb.consume(st,1<<20); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
print("c4 ms", ["%.1f"%t for t in ts], int(sums.sum()))
PY
