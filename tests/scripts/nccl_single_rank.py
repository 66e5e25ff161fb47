"""--force-dist correctness: ShardedLikelihood.eval must equal Evaluator.eval
for alternating variants (a stale read would return the previous result)."""
import os, socket, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, torch.distributed as dist
from paper_2407_11349_b200 import Evaluator, HawkesParams, Variant, benchmark_catalog
from paper_2407_11349_b200.dist import ShardedLikelihood
with socket.socket() as sk:
    sk.bind(("127.0.0.1", 0)); port = sk.getsockname()[1]
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
cat = benchmark_catalog(200000, 42)
sh = ShardedLikelihood(cat, device=0)
ev = Evaluator(cat)
for v in (0, 1, 0, 1):
    p = HawkesParams(mu0=1.0, tau_t=5.0, xi0=0.5, sigma_x=0.5, sigma_t=2.0, area=100.0, variant=Variant(v))
    a = sh.eval(p); b = ev.eval(p, grad=True)
    print(v, a[0], b[0], a[0] == b[0] and (a[1] == b[1]).all(), flush=True)
    assert a[0] == b[0]
dist.destroy_process_group()
