import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import torch.distributed as dist
from cases import training_plan
from test_gpu_distributed_emulated import CopyTransport
from paper_2602_15883_b200.runtime import driver
golden = np.load("tests/golden/golden.npz")
_, plan = training_plan("t2", golden)
dist.get_world_size = lambda *a, **k: plan.n_ranks
tr = CopyTransport(plan)
driver.post_exchange = tr
sms = torch.cuda.get_device_properties(0).multi_processor_count
ts = [driver.DistributedTrainer(plan, rank=r, overlap=True, reserve_sms=sms - 16) for r in range(plan.n_ranks)]
for t in ts:
    t.gate = t.worker.objective.make_gate(t.gate_word, t.worker.flags, timeout_ms=2000)
    tr.register(t)
log = []
def body(t):
    with torch.cuda.stream(torch.cuda.Stream()):
        for e in range(3):
            t.epoch(e)
            torch.cuda.current_stream().synchronize()
            log.append((t.rank, e, int(t.worker.flags.item()), int(t.gate_word.item()), time.time()))
ths = [threading.Thread(target=body, args=(t,)) for t in ts]
[x.start() for x in ths]; [x.join(60) for x in ths]
for l in sorted(log): print(l)
