# in-place consumers: Langevin / gaussian parity + gaussian() per-launch timing at 3..24 deviates per atom
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_langevin.py tests/test_gpu_parity.py -q -x -k "langevin or gaussian or inplace" > gpurun_out/k6_pt.log 2>&1; echo pt=$?; tail -2 gpurun_out/k6_pt.log
timeout 300 python - <<'PY'
import torch, paper_2512_00093_b200 as rb
n=1<<24
st=rb.make_streams(7,2**50,n); g=rb.gauss_states_from(st)
out=torch.empty((8,n,3),dtype=torch.float64,device="cuda")
res=[]
for G in (1,2,4,8):
    gg=g.clone(); rb.gaussian(gg,3,G,out=out[:G]); torch.cuda.synchronize()
    a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    a.record()
    for r in range(10): rb.gaussian(gg,3,G,out=out[:G])
    b.record(); b.synchronize(); res.append("steps=%d %.3f ms/launch" % (G, a.elapsed_time(b)/10))
print(res)
PY
