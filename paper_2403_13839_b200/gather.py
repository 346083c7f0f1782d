"""The optional final gather of a sharded run: every rank's per-root
results -- text offsets, lengths, statuses, error attributes and the flat text
buffer -- collected with torch.distributed collectives on the device tensors
(NCCL over NVLink on GPUs, gloo on CPU tensors in the tests).  It is an
all-gather-v done as padded all-gathers: sizes first, then each array padded to
the largest rank's length.  The result indexes roots in rank order; rank r's text
lives at r * t_max + its own offsets in the gathered text buffer.  There is no
collective on the decompile path itself; this runs after it, and the bench times
it separately."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Gathered:
    text_off: np.ndarray    # uint64, offsets into `text`
    text_len: np.ndarray    # uint32
    status: np.ndarray      # int32
    aux: np.ndarray         # int64 [n, 2]
    text: np.ndarray        # uint8, rank r's bytes at r * t_max
    ranks: list             # (first root, n roots) per rank

    def item(self, i):
        s = self.text[int(self.text_off[i]):int(self.text_off[i]) + int(self.text_len[i])]
        return int(self.status[i]), bytes(s).decode("utf-8", "surrogatepass")


def device_views(meta, text, n):
    """(off, aux, lens, status) views of a DeviceArena meta buffer (layout: api.py
    DeviceArena: [used u64 | pad][off u64 n][aux i64 2n][len u32 n][status i32 n])."""
    import torch

    off = meta[64:64 + 8 * n].view(torch.int64)
    aux = meta[64 + 8 * n:64 + 24 * n].view(torch.int64).view(n, 2)
    lens = meta[64 + 24 * n:64 + 28 * n].view(torch.int32)
    status = meta[64 + 28 * n:64 + 32 * n].view(torch.int32)
    return off, aux, lens, status


def gather_results(off, aux, lens, status, text, group=None) -> Gathered:
    """All-gather the results of every rank.  off/aux/lens/status: this rank's
    per-root tensors (int64 / int64 [n,2] / int32 / int32); text: its uint8 text
    (only the used prefix).  All on the process group's device."""
    import torch
    import torch.distributed as dist

    dev = off.device
    world = dist.get_world_size(group)
    n = int(off.numel())
    sizes = torch.tensor([n, int(text.numel())], dtype=torch.int64, device=dev)
    all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes, group=group)
    ns = [int(s[0]) for s in all_sizes]
    ts = [int(s[1]) for s in all_sizes]
    n_max, t_max = max(max(ns), 1), max(max(ts), 1)
    # one int64 row per root: off, aux0, aux1, len << 32 | status
    rows = torch.zeros((n_max, 4), dtype=torch.int64, device=dev)
    if n:
        rows[:n, 0] = off
        rows[:n, 1:3] = aux
        rows[:n, 3] = (lens.to(torch.int64) << 32) | (status.to(torch.int64) & 0xFFFFFFFF)
    tpad = torch.zeros(t_max, dtype=torch.uint8, device=dev)
    tpad[:text.numel()] = text
    all_rows = [torch.empty_like(rows) for _ in range(world)]
    all_text = [torch.empty_like(tpad) for _ in range(world)]
    dist.all_gather(all_rows, rows, group=group)
    dist.all_gather(all_text, tpad, group=group)
    offs, lens_o, sts, auxs, ranks = [], [], [], [], []
    first = 0
    for r in range(world):
        m = all_rows[r][:ns[r]].cpu().numpy()
        offs.append(m[:, 0].astype(np.uint64) + np.uint64(r * t_max))
        auxs.append(m[:, 1:3].copy())
        lens_o.append((m[:, 3] >> 32).astype(np.uint32))
        sts.append((m[:, 3] & 0xFFFFFFFF).astype(np.uint32).view(np.int32))
        ranks.append((first, ns[r]))
        first += ns[r]
    text_all = torch.cat(all_text).cpu().numpy()
    cat = np.concatenate
    return Gathered(cat(offs) if offs else np.zeros(0, np.uint64), cat(lens_o), cat(sts),
                    cat(auxs) if auxs else np.zeros((0, 2), np.int64), text_all, ranks)
