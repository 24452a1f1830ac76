import sys, time
import torch
sys.path.insert(0, "/root/repo")
import bench
from paper_2403_01444_b200.stage1 import Stage1Config, Stage1Trainer
sc, cache, targets = bench.build_problem(1)
tr = Stage1Trainer(sc.cloud, cache, list(zip(sc.cameras, targets)), Stage1Config())
n = len(sc.cameras)
host_t = [t.cpu().pin_memory() for t in targets]
tr.run_from_host([k % n for k in range(2 * n)], host_t)
tr.reset_frame(); torch.cuda.synchronize()
order = [k % n for k in range(150)]
# instrumented copy of run_from_host: enqueue time vs total
import types
t0 = time.perf_counter()
tr.run_from_host(order, host_t)
t1 = time.perf_counter()
print("run_from_host wall per step ms", (t1 - t0) / 150 * 1e3)
# pure iterate with resident targets, wall clock, same frame window
tr.reset_frame(); torch.cuda.synchronize()
t0 = time.perf_counter()
for k in order:
    tr.iterate(k)
t_enq = time.perf_counter()
torch.cuda.synchronize()
t1 = time.perf_counter()
print("iterate resident: enqueue per step ms", (t_enq - t0) / 150 * 1e3, "wall per step ms", (t1 - t0) / 150 * 1e3)
# host cost of run_from_host pieces: enqueue only (no sync) measured by timing until loop end
main = torch.cuda.current_stream()
tr.reset_frame(); torch.cuda.synchronize()
t0 = time.perf_counter()
for k in order:
    tr.iterate(k, target=tr.targets[k % n])
    tr.loss_dev.to("cpu", non_blocking=True)
t_enq = time.perf_counter()
torch.cuda.synchronize(); t1 = time.perf_counter()
print("iterate+loss D2H: enqueue per step ms", (t_enq - t0) / 150 * 1e3, "wall", (t1 - t0) / 150 * 1e3)
