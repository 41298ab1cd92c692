# gaussian(): parity tests + config-5 timing (2^24 atoms x 3 x 100)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_langevin.py tests/test_gpu_fullsize.py tests/test_gpu_ranmars.py -q -x -k "gaussian or fp64 or config5" > gpurun_out/gk_pt.log 2>&1; echo pt=$?; tail -3 gpurun_out/gk_pt.log
timeout 300 python - <<'PY'
import torch, paper_2512_00093_b200 as rb
n=1<<24
st=rb.make_streams(7,2**50,n); g=rb.gauss_states_from(st)
out=torch.empty((100,n,3),dtype=torch.float64,device="cuda")
rb.gaussian(g.clone(),3,20,out=out[:20]); torch.cuda.synchronize()
ts=[]
for r in range(3):
    gg=g.clone(); torch.cuda.synchronize()
    a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    a.record(); rb.gaussian(gg,3,100,out=out); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
print("config 5 ms", ["%.2f"%t for t in ts], "sum", float(out[99].sum()), int(gg.sum()))
PY
