mkdir -p gpurun_out
for k in 64; do RANMAR_GAUSS_GT=$k timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "gaussian or fp64" > gpurun_out/gk_pt$k.log 2>&1; echo K=$k pt=$?; tail -2 gpurun_out/gk_pt$k.log; done
for k in 32 64 96 128 256; do RANMAR_GAUSS_GT=$k timeout 300 python - <<'PY'
import os, torch, paper_2512_00093_b200 as rb
n=1<<24
st=rb.make_streams(7,2**50,n); g=rb.gauss_states_from(st)
out=torch.empty((100,n,3),dtype=torch.float64,device="cuda")
rb.gaussian(g.clone(),3,2,out=out[:2]); torch.cuda.synchronize()
ts=[]
for r in range(3):
    gg=g.clone(); torch.cuda.synchronize()
    a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    a.record(); rb.gaussian(gg,3,100,out=out); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
print("K", os.environ["RANMAR_GAUSS_GT"], "ms", ["%.2f"%t for t in ts], "sum", float(out[99].sum()), float(out[0].sum()))
PY
done
