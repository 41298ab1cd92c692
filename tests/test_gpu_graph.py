"""The _dev contract (include/ranmar_b200.h): after ranmar_device_setup the
device entry points never allocate, synchronise or read device memory back,
so a fresh process can capture them in a CUDA graph and replay it bit-exactly
(checked against the oracle). Runs in a subprocess so the device really is
fresh (no earlier test set it up)."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import ctypes, sys
import numpy as np, torch
sys.path.insert(0, ROOT)
import paper_2512_00093_b200 as rb
from oracle.bind import Oracle
torch.cuda.set_device(0)
L = rb.lib()
n, per = 300, 4103
states = torch.empty((n, 100), dtype=torch.int32, device="cuda")
out = torch.empty(n * per, dtype=torch.float32, device="cuda")
# before ranmar_device_setup: the _dev entry points refuse (RANMAR_ESTATE = 4)
assert L.ranmar_generate_f32_dev(ctypes.c_void_p(states.data_ptr()), n, per,
                                 ctypes.c_void_p(out.data_ptr()), None) == 4
rb.device_setup(0)
base = rb.init(12345)
ws = torch.empty(L.ranmar_make_streams_workspace(n), dtype=torch.uint8, device="cuda")
one = torch.from_numpy(base.view(np.int32).reshape(1, 100).copy()).cuda()
count1 = 10**6
out1 = torch.empty(count1, dtype=torch.float32, device="cuda")
ws1 = torch.empty(int(L.ranmar_generate_single_workspace(count1)), dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):   # global capture mode: any sync or malloc would fail
    rb.make_streams_dev(base, 2**40, n, out=states, workspace=ws, stream=s)
    rb.generate(states, per, "f32", out=out, stream=s)
    rc = L.ranmar_generate_single_f32_dev(ctypes.c_void_p(one.data_ptr()), count1,
                                          ctypes.c_void_p(out1.data_ptr()), ctypes.c_void_p(ws1.data_ptr()),
                                          ws1.numel(), ctypes.c_void_p(s.cuda_stream))
    assert rc == 0, L.ranmar_last_error()
launches = rb.kernel_launches()
g.replay()
torch.cuda.synchronize()
assert rb.kernel_launches() == launches   # replays launch nothing through the host library
orc = Oracle()
es = orc.make_streams(orc.init(12345), 2**40, n)
exp = orc.generate_f32(es, per)
assert (out.cpu().numpy() == exp).all()
assert rb.states_to_host(states).tobytes() == es.tobytes()
os1 = orc.init(12345)
e1 = orc.generate_f32(os1, count1)
assert (out1.cpu().numpy() == e1).all() and rb.states_to_host(one).tobytes() == os1.tobytes()
a, a1 = out.clone(), out1.clone()
g.replay()   # make_streams rewrites the states: the same outputs again; the single stream moves on
torch.cuda.synchronize()
assert torch.equal(a, out)
e2 = orc.generate_f32(os1, count1)
assert (out1.cpu().numpy() == e2).all() and rb.states_to_host(one).tobytes() == os1.tobytes()
assert rb.device_status() == 0
print("graph replay bit-exact")
'''


def test_dev_calls_capture_in_a_cuda_graph_on_a_fresh_device():
    r = subprocess.run([sys.executable, "-c", f"ROOT = {ROOT!r}\n" + SCRIPT], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "graph replay bit-exact" in r.stdout
