import math, time, sys, subprocess, threading, numpy as np, torch
sys.path.insert(0, '.')
import paper_2009_14788_b200 as rk
from paper_2009_14788_b200.phantom import shepp_logan
ga = rk.make_parallel(512, [(i * 100.0 / 512 - 50.0) * math.pi / 180.0 for i in range(512)])
op = rk.projector_operator(ga)
plan = rk.make_plan(512, 512, [0.5] * 5)
x = torch.from_numpy(np.stack([shepp_logan(512)] * 8)).cuda()
clk = []
stop = False
def sampler():
    while not stop:
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active", "--format=csv,noheader"], capture_output=True, text=True)
        clk.append(r.stdout.strip()); time.sleep(0.2)
th = threading.Thread(target=sampler); th.start()
for b in (1, 8):
    y = rk.forward(ga, x[:b])
    for run in range(6):
        free0 = torch.cuda.mem_get_info()[0]
        torch.cuda.synchronize(); a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n0 = len(clk); a.record()
        rk.admm_reconstruct(op, plan, y, rk.AdmmParams(outer_iterations=50, inner_cg_iterations=50))
        e.record(); torch.cuda.synchronize()
        print(f"b={b} run {run}: {a.elapsed_time(e):.0f} ms, free mem {free0/1e9:.2f} GB, clocks {sorted(set(clk[n0:]))[:3]}", flush=True)
stop = True; th.join()
