import sys, ctypes as C, numpy as np, torch
sys.argv=['bench.py','--steps','3','--warmup','1','--no-cpu-baseline','--e2e-steps','0']
import bench
from paper_2511_14617_b200 import _lib
L=_lib.lib()
L.dgds_debug_query_timing.argtypes=[C.c_void_p, C.c_void_p]
orig = _lib.lib().dgds_speculate_device
buf = torch.zeros((65536, 8), dtype=torch.int64, device='cuda:0')
state = {'set': False}
import paper_2511_14617_b200.dgds as D
_orig_update = D.DraftServer.update_device
def upd(self, *a, **k):
    if not state['set']:
        L.dgds_debug_query_timing(self.handle, C.c_void_p(buf.data_ptr())); state['set']=True
    return _orig_update(self, *a, **k)
D.DraftServer.update_device = upd
bench.main()
torch.cuda.synchronize()
d = buf.cpu().numpy()
d = d[d[:,0] > 0]
print('queries', len(d))
for i, name in enumerate(['phaseA_cyc','phaseB_cyc','out_cyc','depth_it','child_it','merge_it','winner','nf']):
    v = d[:, i]
    print(f'{name:12s} mean {v.mean():10.1f} p50 {np.percentile(v,50):10.1f} p90 {np.percentile(v,90):10.1f} max {v.max()}')
