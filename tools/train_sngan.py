"""SN-GAN 128x128 class-conditional training step with cross-replica BatchNorm
(BASELINE.json configs[3]).

Generator (SAGAN/BigGAN-style, the survey's 11 cross-replica BN layers, SURVEY.md
§8a): z(120) + class embedding -> 4x4x1024 -> five up-sampling residual blocks
1024->1024->512->256->128->64 at 8..128 px, each BN(cin) -> ReLU -> nearest x2 ->
conv3x3 -> BN(cout) -> ReLU -> conv3x3 plus an up-sampled 1x1 shortcut, then
BN(64) -> ReLU -> conv3x3 -> tanh: BN widths 1024, 1024, 1024, 512, 512, 256, 256,
128, 128, 64, 64. Every BN in the generator is the per-channel cross-replica BN of
this repo (K5 forward statistics, K5b backward statistics over NVLink).
Discriminator: spectrally normalised conv stack with a projection head (hinge
loss). Both optimizers (Adam, PAPER.md:296's SN-GAN hyper-parameters) are wrapped.
Synthetic data; global batch = 64 x N
(PAPER.md:285). The builder's channel plan follows SURVEY.md §8a.

  torchrun --nproc-per-node N tools/train_sngan.py
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.nn as nn  # noqa: E402
import torch.nn.functional as F  # noqa: E402

SN = nn.utils.spectral_norm
CH = [1024, 1024, 512, 256, 128, 64]  # 4 -> 128 px


class GBlock(nn.Module):
    """Residual up-sampling block with two cross-replica BNs (BN(cin), BN(cout))."""

    def __init__(self, cin, cout, repl, bn_cls):
        super().__init__()
        self.bn1, self.bn2 = bn_cls(cin, repl), bn_cls(cout, repl)
        self.conv1 = nn.Conv2d(cin, cout, 3, padding=1)
        self.conv2 = nn.Conv2d(cout, cout, 3, padding=1)
        self.skip = nn.Conv2d(cin, cout, 1)

    def forward(self, x):
        h = F.interpolate(F.relu(self.bn1(x)), scale_factor=2, mode="nearest")
        h = self.conv2(F.relu(self.bn2(self.conv1(h))))
        return h + self.skip(F.interpolate(x, scale_factor=2, mode="nearest"))


class Generator(nn.Module):
    def __init__(self, repl, nz=120, ncls=1000, bn_cls=None):
        super().__init__()
        self.embed = nn.Embedding(ncls, nz)
        self.fc = nn.Linear(2 * nz, 4 * 4 * CH[0])
        self.blocks = nn.ModuleList([GBlock(a, b, repl, bn_cls) for a, b in zip(CH[:-1], CH[1:])])
        self.bn_out = bn_cls(CH[-1], repl)
        self.out = nn.Conv2d(CH[-1], 3, 3, padding=1)

    def forward(self, z, y):
        h = self.fc(torch.cat([z, self.embed(y)], 1)).view(-1, CH[0], 4, 4)
        h = h.contiguous(memory_format=torch.channels_last)
        for blk in self.blocks:
            h = blk(h)
        return torch.tanh(self.out(F.relu(self.bn_out(h))))


class Discriminator(nn.Module):
    def __init__(self, ncls=1000):
        super().__init__()
        chs = [3, 64, 128, 256, 512, 1024, 1024]
        self.convs = nn.ModuleList([SN(nn.Conv2d(a, b, 4, stride=2, padding=1)) for a, b in zip(chs[:-1], chs[1:])])
        self.fc = SN(nn.Linear(chs[-1], 1))
        self.embed = SN(nn.Embedding(ncls, chs[-1]))

    def forward(self, x, y):
        h = x
        for c in self.convs:
            h = F.leaky_relu(c(h), 0.2)
        h = h.sum(dim=(2, 3))
        return self.fc(h).squeeze(1) + (self.embed(y) * h).sum(1)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--batch", type=int, default=64)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    a = p.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    from paper_1902_00465_b200 import CrossReplicaBatchNorm, Replicator

    torch.backends.cudnn.benchmark = True
    repl = Replicator(device=local, pool_bytes=512 << 20)
    torch.manual_seed(rank)
    with repl.context():
        G = repl.replicate(lambda: Generator(repl, bn_cls=CrossReplicaBatchNorm).to(memory_format=torch.channels_last))
        D = repl.replicate(lambda: Discriminator().to(memory_format=torch.channels_last))
        g_opt = repl.wrap_optimizer(torch.optim.Adam(G.parameters(), lr=1e-4, betas=(0.0, 0.999)))
        d_opt = repl.wrap_optimizer(torch.optim.Adam(D.parameters(), lr=4e-4, betas=(0.0, 0.999)))
    gen = torch.Generator(device=dev).manual_seed(100 + rank)
    real = (torch.rand(a.batch, 3, 128, 128, device=dev, generator=gen) * 2 - 1).contiguous(
        memory_format=torch.channels_last)
    yr = torch.randint(0, 1000, (a.batch,), device=dev, generator=gen)

    def step():
        z = torch.randn(a.batch, 120, device=dev, generator=gen)
        yf = torch.randint(0, 1000, (a.batch,), device=dev, generator=gen)
        with torch.autocast("cuda", dtype=torch.bfloat16):
            fake = G(z, yf)
            d_loss = F.relu(1 - D(real, yr)).mean() + F.relu(1 + D(fake.detach(), yf)).mean()
        d_opt.zero_grad(set_to_none=False)
        d_loss.backward()
        d_opt.step()
        with torch.autocast("cuda", dtype=torch.bfloat16):
            g_loss = -D(G(z, yf), yf).mean()
        g_opt.zero_grad(set_to_none=False)
        g_loss.backward()
        g_opt.step()
        return d_loss, g_loss

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    st = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(a.steps):
        dl, gl = step()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = t.item()
    # the cross-replica BN statistics must be identical on every replica
    rm = torch.cat([b.running_mean for b in G.local.bns])
    gathered = repl.all_gather(rm, stack=True) if world > 1 else rm.unsqueeze(0)
    same = bool(all(torch.equal(gathered[r], gathered[0]) for r in range(world)))
    if rank == 0:
        print(json.dumps({"metric": "SN-GAN step (D+G) img/s", "value": world * a.batch / (ms / 1e3), "unit": "img/s",
                          "n_gpus": world, "per_gpu_batch": a.batch, "ms_per_step": ms,
                          "d_loss": float(dl.item()), "g_loss": float(gl.item()),
                          "bn_running_stats_identical": same,
                          "config": {"resolution": 128, "generator_bn": "CrossReplicaBatchNorm x11 (K5/K5b; widths 1024x3, 512x2, 256x2, 128x2, 64x2)",
                                     "precision": "bf16 autocast", "data": "synthetic"}}), flush=True)
    repl.comm.close()
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
