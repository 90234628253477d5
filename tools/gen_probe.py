import sys, time, torch
sys.path.insert(0, '/root/repo')
import gcp_synth
t0 = time.time()
def log(*a): print(f"[{time.time()-t0:7.1f}s]", *a, file=sys.stderr, flush=True)
c = gcp_synth.CONFIGS['c4']
n = int(sys.argv[1]) if len(sys.argv) > 1 else c['nnz']
log("start", n)
s, v = gcp_synth.chi_kolda(c['dims'], n, c['R'], 1004, c['loss'], device='cuda')
torch.cuda.synchronize(); log("generated", s.shape, torch.cuda.max_memory_allocated()/1e9, "GB peak")
sh = s.cpu(); log("to cpu subs")
sp = sh.pin_memory(); log("pinned subs")
