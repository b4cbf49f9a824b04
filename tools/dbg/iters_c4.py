import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2306_08152_b200 as qf, qfgen
w = qfgen.workload("C4")
c = qf.Circuit.from_workload(w)
r = qf.qf_instantiate(c, w.target_unitary(), None, num_starts=w.starts, seed=w.init_seed, max_iters=w.max_iters)
it = r.iters
print("iters min/mean/max", it.min(), it.mean(), it.max(), "p50/p90/p99", np.percentile(it, [50, 90, 99]))
# greedy schedule with 444 slots in start order, durations proportional to iters
import heapq
slots = [0.0] * 444
heapq.heapify(slots)
for d in it:
    t = heapq.heappop(slots); heapq.heappush(slots, t + d)
mk = max(slots); ideal = it.sum() / 444
print("makespan/ideal", mk / ideal)
