"""Desk-scale PETRA training with the paper's recipe.

Recipe: SGD with Nesterov momentum 0.9; weight decay 5e-4 on CIFAR-10,
none on the BN parameters and biases; batch 64 with gradient accumulation k (the average
of the accumulated gradients) and base learning rate lr = 0.1 * 64k / 256; a linear
warm-up from 0 over the first 5 of 300 epochs, then x0.1 at epochs 150 and 225 -- the
same fractions of a shorter run here.  The running statistics of BN are updated during
the backward recomputation and used for evaluation (petra_stage_eval).
J = 1 is plain backpropagation through the same library (one stage: forward, loss,
backprop and update in one tick, the oracle's J = 1 == backprop pin).

The data is synthetic (no network here for CIFAR-10): `synth_images` draws a seeded,
class-conditional Gaussian 3x32x32 task with the paper's augmentation
(random 4-pixel-padded crops, horizontal flips).  A test set is
drawn from the same distribution with other seeds.  PyTorch only generates data and
holds buffers; every step of training runs in libpetra.
"""
from __future__ import annotations

import math

import torch

from . import _lib as L
from . import models as PM
from .petra import Pipeline


def synth_images(n, classes=10, seed=0, sigma=1.0, sep=3.0, device="cuda", augment=True):
    """n seeded images [n, 32, 32, 3] (NHWC, fp32) and labels int32[n]: class-conditional
    Gaussians -- x = mu_y + sigma * N(0, I) with smooth class templates mu_c
    (8x8x3 Gaussian draws upsampled bilinearly, scaled so that the templates lie about
    `sep` sigma apart), so the Bayes accuracy is below 100 % and a gap between training
    methods is measurable."""
    g = torch.Generator(device=device).manual_seed(seed)
    y = torch.randint(0, classes, (n,), generator=g, device=device)
    gc = torch.Generator(device=device).manual_seed(12345)  # the task's templates: fixed
    t = torch.randn(classes, 3, 8, 8, generator=gc, device=device)
    t = torch.nn.functional.interpolate(t, size=(32, 32), mode="bilinear", align_corners=False)
    t = t / t.flatten(1).norm(dim=1)[:, None, None, None] * (sep * sigma / math.sqrt(2.0))
    img = t[y].permute(0, 2, 3, 1) + sigma * torch.randn((n, 32, 32, 3), generator=g, device=device)
    if augment:  # random crop of the 4-pixel zero-padded image, horizontal flip
        pad = torch.nn.functional.pad(img.permute(0, 3, 1, 2), (4, 4, 4, 4))
        ox = torch.randint(0, 9, (n,), generator=g, device=device)
        oy = torch.randint(0, 9, (n,), generator=g, device=device)
        ar = torch.arange(32, device=device)
        rows = (oy[:, None] + ar[None])[:, None, :, None].expand(n, 3, 32, 40)
        img = torch.gather(pad, 2, rows)
        cols = (ox[:, None] + ar[None])[:, None, None, :].expand(n, 3, 32, 32)
        img = torch.gather(img, 3, cols).permute(0, 2, 3, 1)
        flip = torch.rand(n, generator=g, device=device) < 0.5
        img = torch.where(flip[:, None, None, None], img.flip(2), img)
    return img.contiguous(), y.to(torch.int32)


def lr_schedule(epoch: float, base: float, epochs: int):
    """Linear warm-up over the first 5/300 of the run, x0.1 at 1/2 and 3/4."""
    warm = max(1.0, epochs * 5.0 / 300.0)
    if epoch < warm:
        return base * epoch / warm
    return base * (0.1 ** ((epoch >= epochs * 0.5) + (epoch >= epochs * 0.75)))


def evaluate(pipe: Pipeline, J, x, y, batch, classes):
    """Test accuracy and mean loss through petra_stage_eval (BN on the running statistics)."""
    dev = x.device
    correct = torch.zeros(1, dtype=torch.int32, device=dev)
    loss = torch.zeros(1, device=dev)
    tot_loss, nb = 0.0, 0
    bufs = {}
    for b0 in range(0, x.shape[0] - batch + 1, batch):
        cur = [x[b0:b0 + batch].contiguous(), None]
        for j in range(1, J + 1):
            s = pipe.stages[j]
            if j == J:
                s.eval_tail(cur[0], cur[1], y[b0:b0 + batch].contiguous(), correct, loss)
            else:
                if j not in bufs:
                    bufs[j] = [torch.empty(s.out_shape, device=dev) for _ in range(2)]
                s.eval(cur[0], cur[1], bufs[j][0], bufs[j][1])
                cur = bufs[j]
        torch.cuda.synchronize()
        tot_loss += loss.item()
        nb += 1
    return correct.item() / (nb * batch), tot_loss / max(nb, 1)


def train(model="revnet18", J=4, k=1, epochs=12, n_train=25600, n_test=2560, batch=64, classes=10,
          precision=L.BF16_TC, seed=0, sigma=1.0, log=None):
    """Train `model` with PETRA over J stages (J = 1: backpropagation) on the synthetic task;
    returns a dict with the per-epoch train loss and the final test accuracy / loss."""
    torch.cuda.set_device(0)
    units = PM.revnet(model, 32, classes)
    counts = [len(units)] if J == 1 else PM.partition(units, J, batch, 32, 32, 3)
    specs = PM.stage_specs(units, counts, batch, (32, 32, 3), precision, 5e-4, accumulation_k=k)
    pipe = Pipeline(specs, [0] * J, 0, 1, seed=seed + 1)
    base = 0.1 * 64 * k / 256
    steps = n_train // batch
    xt, yt = synth_images(n_test, classes, seed=10_000 + seed, sigma=sigma, augment=False)
    loss = torch.zeros(1, device="cuda")
    hist, t = [], 0
    for ep in range(epochs):
        x, y = synth_images(steps * batch, classes, seed=seed * 1000 + ep, sigma=sigma)
        acc_loss, n_loss = 0.0, 0
        for i in range(steps):
            lr = lr_schedule(ep + i / steps, base, epochs)
            pipe.tick(t, True, x[i * batch:(i + 1) * batch], y[i * batch:(i + 1) * batch], lr, loss, report=False)
            t += 1
            if i % 16 == 15:
                torch.cuda.synchronize()
                acc_loss += loss.item()
                n_loss += 1
        hist.append(acc_loss / max(n_loss, 1))
        if log:
            log(f"J={J} k={k} epoch {ep + 1}/{epochs} lr {lr:.4f} train loss {hist[-1]:.4f}")
    for _ in range(2 * J - 2):  # drain: the last micro-batches' backwards and updates
        pipe.tick(t, False, None, None, lr_schedule(epochs, base, epochs), loss, report=False)
        t += 1
    torch.cuda.synchronize()
    acc, tl = evaluate(pipe, J, xt, yt, batch, classes)
    pipe.close()
    return {"model": model, "J": J, "k": k, "partition": counts, "epochs": epochs, "n_train": steps * batch,
            "n_test": n_test, "batch": batch, "base_lr": base, "train_loss": hist, "test_accuracy": acc,
            "test_loss": tl, "ticks": t}
