import torch, sys
sys.path.insert(0, '/root/repo')
import paper_2512_00093_b200 as rb
st=rb.make_streams_dev(rb.init_unchecked(987654321),2**120,1<<20)
for r in range(3):
    t,o=rb.to_text_dev(st); s2,e=rb.from_text_dev(t,o)
torch.cuda.synchronize()
