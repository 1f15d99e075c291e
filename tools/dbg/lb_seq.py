"""Debug: random sequence of collectives in a loopback world (W ranks on one GPU), each
checked against the oracle. PINNED=1 copies results through pinned memory (the
product path, comm.to_host); CHECK=1 adds comm.check() after every op."""
import os, sys
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "backend:cudaMallocAsync")
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
from paper_1902_00465_b200.bootstrap import LoopbackWorld
from paper_1902_00465_b200.comm import Communicator
from oracle import collectives as O

W = int(os.environ.get("W", "2"))
N = int(os.environ.get("N", "40"))
POOL = int(os.environ.get("POOL", str(32 << 20)))
rng = np.random.default_rng(int(os.environ.get("SEED", "0")))
ops = []
for i in range(N):
    op = rng.choice(["ar", "ar_inplace", "ar_pool", "ag", "bc"])
    count = int(rng.choice([1, 7, 1000, 4097, 65536, 203530, 262144]))
    ops.append((op, count, i))
print(len(ops), "ops", flush=True)

def body(rank):
    pinned = torch.empty(8 << 20, dtype=torch.float32, pin_memory=True) if os.environ.get("PINNED") else None

    def host(t):
        if pinned is None:
            return t.cpu().numpy()
        n = t.numel()
        if os.environ.get("PINNED") == "2":  # a fresh pinned allocation per copy
            h = torch.empty(n + int(np.random.randint(1, 1 << 20)), dtype=torch.float32, pin_memory=True)[:n]
        else:
            h = pinned[:n]
        h.copy_(t.reshape(-1), non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return h.numpy().copy().reshape(t.shape)
    comm = Communicator(device=0, bootstrap=lw.bootstrap(rank), pool_bytes=POOL, timeout_s=float(os.environ.get("TMO", "5")))
    bucket = comm.alloc(300000, torch.float32)
    log = []
    import time
    T0 = time.time()
    for op, count, i in ops:
        t_start = time.time() - T0
        xs = [np.random.default_rng(1000 * i + r).standard_normal(count).astype(np.float32) for r in range(W)]
        x = torch.from_numpy(xs[rank]).cuda()
        if op == "ar":
            got = host(comm.all_reduce_tensor(x, "sum")); want = O.fold_sum(xs)
        elif op == "ar_inplace":
            comm.all_reduce_tensor(x, "sum", out=x); got = host(x); want = O.fold_sum(xs)
        elif op == "ar_pool":
            b = bucket[:count]; b.copy_(x); comm.all_reduce_tensor(b, "premean", out=b)
            got = host(b); want = O.fold_premean(xs)
        elif op == "ag":
            got = host(comm.all_gather_tensor(x)).reshape(-1); want = np.concatenate(xs)
        else:
            comm.broadcast_tensor(x, root=i % W); got = host(x); want = xs[i % W]
        t_got = time.time() - T0
        st = ""
        if os.environ.get("CHECK"):
            try:
                comm.check(); st = "ok"
            except Exception as e:
                st = "ABORT " + str(e)[60:300]
        bad = int((got.view(np.uint32) != want.view(np.uint32)).sum())
        t_chk = time.time() - T0
        st = st + f" t={t_start:.3f}/{t_got:.3f}/{t_chk:.3f}"
        log.append((i, op, count, bad, st))
        if os.environ.get("VERBOSE"):
            print("rank", rank, (i, op, count, bad, st), flush=True)
    try:
        comm.check()
    except Exception as e:
        log.append(("final", str(e)[:200]))
    comm.close()
    return log

lw = LoopbackWorld(W, device=0)
out = lw.run(body)
nbad = 0
for r, log in enumerate(out):
    for row in log:
        if row[0] == "final" or row[3] or "ABORT" in row[4]:
            nbad += 1
            print("rank", r, row, flush=True)
print("bad rows:", nbad)
sys.exit(1 if nbad else 0)
