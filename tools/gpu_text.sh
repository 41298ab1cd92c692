mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_text.py tests/test_cli.py -q -x > gpurun_out/tx_pt.log 2>&1; echo pt=$?; tail -2 gpurun_out/tx_pt.log
timeout 300 python - <<'PY'
import torch, paper_2512_00093_b200 as rb
n=1<<20
st=rb.make_streams_dev(rb.init_unchecked(987654321),2**120,n)
text,off=rb.to_text_dev(st); torch.cuda.synchronize()
ts=[];tf=[]
for r in range(5):
    a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True); c=torch.cuda.Event(enable_timing=True)
    a.record(); text,off=rb.to_text_dev(st); b.record(); s2,err=rb.from_text_dev(text,off); c.record(); c.synchronize()
    ts.append(a.elapsed_time(b)); tf.append(b.elapsed_time(c))
print("to_text ms", ["%.2f"%x for x in ts], "from_text ms", ["%.2f"%x for x in tf], int(off[-1]), bool(torch.equal(s2,st)), int(err.abs().sum()))
PY
