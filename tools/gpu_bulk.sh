# make_streams: parity tests + config 3 (2^20 stream starts at J = 2^120)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "make_streams or config3 or config4_full or jump or config2_full or beyond" > gpurun_out/bulk_pt.log 2>&1; echo pt=$?; tail -3 gpurun_out/bulk_pt.log
timeout 300 python - <<'PY'
import torch, paper_2512_00093_b200 as rb
n=1<<20
st=torch.empty((n,100),dtype=torch.int32,device="cuda")
ws=torch.empty(rb.lib().ranmar_make_streams_workspace(n),dtype=torch.uint8,device="cuda")
b=rb.init_unchecked(987654321)
for _ in range(3): rb.make_streams_dev(b,2**120,n,out=st,workspace=ws)
torch.cuda.synchronize(); ts=[]
for r in range(5):
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record(); rb.make_streams_dev(b,2**120,n,out=st,workspace=ws); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
print("config 3 ms", ["%.3f"%t for t in ts], int(st.sum()))
PY
