import os, sys, time, ctypes, statistics, torch
sys.path.insert(0, '/root/repo')
import paper_2409_14222_b200 as V
from paper_2409_14222_b200.pack import read_pack
from paper_2409_14222_b200.solver import mg_rhs
pack = read_pack('/root/repo/data/cfg2_pack.npz')
hier = V.hierarchy_from_pack(pack)
b = torch.from_numpy(mg_rhs(pack)).cuda()
for _ in range(3): hier.vcycle_device(b)
torch.cuda.synchronize()
g = list(hier._graphs.values())[0]
# host time of g.replay()
ts = []
for _ in range(50):
    t0 = time.perf_counter(); g.replay(); t1 = time.perf_counter(); ts.append(t1 - t0)
    torch.cuda.synchronize()
print("torch replay host us", statistics.median(ts) * 1e6)
# raw cudaGraphLaunch via the library torch loaded
import glob
cands = [p for p in glob.glob(os.path.join(os.path.dirname(torch.__file__), 'lib', 'libcudart*'))] + glob.glob('/usr/local/cuda/lib64/libcudart.so*')
print(cands[:3])
rt = ctypes.CDLL(cands[0])
execp = ctypes.c_void_p(g.raw_cuda_graph_exec())
stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
ts = []
for _ in range(50):
    t0 = time.perf_counter(); e = rt.cudaGraphLaunch(execp, stream); t1 = time.perf_counter(); ts.append(t1 - t0)
    assert e == 0, e
    torch.cuda.synchronize()
print("raw cudaGraphLaunch host us", statistics.median(ts) * 1e6)
# bubble: time from sync return to GPU start: measure back-to-back replays with sync between
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record(); g.replay(); ev1.record(); torch.cuda.synchronize(); print("graph device ms", ev0.elapsed_time(ev1))
