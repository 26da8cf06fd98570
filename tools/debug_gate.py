import os, sys, time
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import torch
from test_gpu_contracts import _small_plan
from paper_2602_15883_b200.runtime.driver import LocalTrainer
_, plan = _small_plan(epochs=2)
tr = LocalTrainer(plan, overlap=True, signal_delay_ns=300_000_000, exchange_timeout=0.02)
for r, g in tr.gate_args.items():
    print(r, g.gate, g.first_gated_set, g.max_ctas, g.flags, g.timeout_ms)
t0 = time.time()
try:
    times = tr.run(1)
    print("times", times)
except Exception as e:
    print("raised", type(e), e)
print("wall", time.time() - t0)
print({r: int(w.flags.item()) for r, w in tr.workers.items()})
