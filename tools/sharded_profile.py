"""cProfile of one world-1 sharded cfg2 factorization (host-side costs)."""
import cProfile, os, pstats, socket, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
import bench
import paper_1509_06820_b200 as P
from paper_1509_06820_b200.parallel import BlockCyclic, rqrcp_sharded
with socket.socket() as s:
    s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]
os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(port)
dev = torch.device("cuda", 0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
cfg = bench.CONFIGS["cfg2"]
A = bench.device_matrix(cfg["kind"], cfg["m"], cfg["n"], dev, seed=0)
cfgP = P.RandomizedConfig(block=cfg["block"], padding=cfg["padding"], seed=0)
rqrcp_sharded(A, cfg["m"], cfg["n"], cfg["k"], cfgP, gather_r=False)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
rqrcp_sharded(A, cfg["m"], cfg["n"], cfg["k"], cfgP, gather_r=False)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
dist.destroy_process_group()
