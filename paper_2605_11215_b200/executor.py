"""Canonical microbatch executor: optimizer steps of a torch module over a
data-parallel replica group, committed by ``GradientCommit``.

The reference trains a toy model whose replica r consumes its own stream
slice (trainer.py:134-168, 202-229), so a failure run commits *different*
examples than the failure-free run and equivalence is only statistical
(test_acceptance.py:227-259).  Here the data of step t's microbatch m is a
pure function of (t, m) — canonical addressing — and the
committed gradient is the canonical tree over m (commit.py).  Survivors
recompute exactly the microbatches the dead replica had not committed; the
ones they already computed are kept.  With deterministic per-microbatch
forward/backward, the loss and parameter trajectory under any failure
schedule is then bitwise the failure-free one.

Parameters live in one flat fp32 buffer (the module's parameters are views
into it) and the committed gradient buffer of replica 0 is the optimizer's
gradient.  Microbatch gradients reach the commit one of two ways:

* ``kacc=True`` (default): backward's per-parameter gradient tensors are
  pushed, in place, into the replica's K-ACC stack (kacc.py): one launch per
  microbatch merges the carry chain, nothing is copied into a flat buffer,
  and a replica holds O(log G) gradient-sized nodes; the commit evaluates the
  top of the canonical tree over the nodes;
* ``kacc=False``: each microbatch gradient is copied into its own flat slot
  (B slots resident) and the commit reads every slot.

Both commit the same bits (the canonical tree depends only on the leaves).
"""

from __future__ import annotations

from typing import Callable, Dict, List, Tuple

import torch
import torch.nn as nn

from . import kacc as _kacc
from .commit import CommitOutcome, GradientCommit


def flatten_module(module: nn.Module, device) -> Tuple[torch.Tensor, List[torch.Tensor]]:
    """Move every trainable parameter of `module` into one flat fp32 buffer;
    returns (flat, params) with each parameter's data now a view of `flat`."""
    params = [p for p in module.parameters() if p.requires_grad]
    numel = sum(p.numel() for p in params)
    flat = torch.empty(numel, dtype=torch.float32, device=device)
    views, off = [], 0
    for p in params:
        v = flat[off:off + p.numel()].view_as(p)
        v.copy_(p.detach().to(device=device, dtype=torch.float32))
        p.data = v
        views.append(v)
        off += p.numel()
    return flat, params


class CanonicalExecutor:
    """Run optimizer steps: every replica computes the canonical microbatches
    the engine assigns to it, the engine commits the canonical tree / B into
    every live replica's gradient, SGD applies it.

    batch_fn(t, m) -> input batch of step t's microbatch m (deterministic);
    loss_fn(module, batch) -> scalar loss.  Replicas of one process share the
    module (their parameters are identical by construction, as the reference
    asserts, trainer.py:451-453)."""

    def __init__(self, module: nn.Module, batch_fn: Callable, loss_fn: Callable,
                 w_init: int, g_init: int, k_buckets: int, lr: float = 0.05,
                 device="cuda:0", spares: int = 0, policy_kind: str = "static",
                 kacc: bool = True):
        self.device = torch.device(device)
        self.module = module.to(self.device)
        self.flat, self.params = flatten_module(self.module, self.device)
        self.numel = self.flat.numel()
        self.engine = GradientCommit(self.numel, w_init, g_init, k_buckets,
                                     placement={r: self.device for r in range(w_init + spares)},
                                     spares=spares, policy_kind=policy_kind)
        self.b = w_init * g_init
        self.g = g_init
        self.kacc = kacc
        if kacc:
            bad = [tuple(p.shape) for p in self.params if p.numel() % 4]
            if bad:
                raise ValueError("K-ACC needs parameters of whole 4-element vectors: %s" % bad[:4])
            self.pool = _kacc.SlotPool(self.numel, self.device)
            self.accs = {r: _kacc.KAccumulator(self.pool) for r in range(w_init + spares)}
        else:
            self.slots = torch.empty(self.b, self.numel, dtype=torch.float32, device=self.device)
        self.batch_fn, self.loss_fn, self.lr = batch_fn, loss_fn, lr
        self.computed: List[Tuple[int, int, int]] = []  # (step, m, rid) forward/backward log

    def _grad_into(self, slot: torch.Tensor, batch) -> torch.Tensor:
        loss = self.loss_fn(self.module, batch)
        grads = torch.autograd.grad(loss, self.params)
        off = 0
        for g in grads:
            n = g.numel()
            slot[off:off + n].copy_(g.reshape(-1))
            off += n
        return loss.detach()

    def memory_report(self) -> dict:
        """K-ACC slot usage against the O(log G) bound (bytes per slot)."""
        if not self.kacc:
            return {"slot_bytes": self.numel * 4, "slots_allocated": self.b}
        return _kacc.memory_report({self.device: self.pool}, self.accs, self.g, self.numel)

    def step(self, t: int, injector=None) -> Tuple[CommitOutcome, float]:
        done: Dict[int, Tuple[int, object]] = {}
        losses: Dict[int, torch.Tensor] = {}
        if self.kacc:
            for acc in self.accs.values():
                acc.reset()

        def leaf(m: int, rid: int):
            # a microbatch is computed once by the replica that admits it; a
            # survivor that takes over a dead replica's index recomputes it
            if m not in done or done[m][0] != rid:
                batch = self.batch_fn(t, m)
                if self.kacc:
                    loss = self.loss_fn(self.module, batch)
                    grads = torch.autograd.grad(loss, self.params)
                    self.accs[rid].push(m, [g.reshape(-1) for g in grads])
                    losses[m] = loss.detach()
                    done[m] = (rid, _kacc.Pending(self.accs[rid], m))
                else:
                    losses[m] = self._grad_into(self.slots[m], batch)
                    done[m] = (rid, self.slots[m])
                self.computed.append((t, m, rid))
            return done[m][1]

        out = self.engine.step(t, leaf, injector)
        committed = sorted(i for v in out.admitted.values() for i in v)
        # committed loss in canonical index order (a fixed left fold)
        loss = torch.zeros((), dtype=torch.float32, device=self.device)
        for m in committed:
            loss = loss + losses[m]
        loss = float(loss) / max(1, len(committed))
        grad = self.engine.grads[self.engine.comm.members[0]]
        with torch.no_grad():
            self.flat.sub_(grad, alpha=self.lr)
        return out, loss


class TinyTransformer(nn.Module):
    """A small causal transformer LM (the "tiny transformer" of BASELINE
    configs[0]); plain matmul attention, so every kernel is deterministic
    under torch.use_deterministic_algorithms."""

    def __init__(self, vocab: int = 256, d: int = 128, heads: int = 4,
                 layers: int = 2, seq: int = 64):
        super().__init__()
        self.heads, self.seq = heads, seq
        self.tok = nn.Embedding(vocab, d)
        self.pos = nn.Parameter(torch.randn(seq, d) * 0.02)
        self.blocks = nn.ModuleList()
        for _ in range(layers):
            self.blocks.append(nn.ModuleDict(dict(
                ln1=nn.LayerNorm(d), qkv=nn.Linear(d, 3 * d), proj=nn.Linear(d, d),
                ln2=nn.LayerNorm(d), fc=nn.Linear(d, 4 * d), out=nn.Linear(4 * d, d))))
        self.ln = nn.LayerNorm(d)
        self.head = nn.Linear(d, vocab, bias=False)
        mask = torch.full((seq, seq), float("-inf")).triu(1)
        self.register_buffer("mask", mask, persistent=False)

    def forward(self, idx: torch.Tensor) -> torch.Tensor:
        b, s = idx.shape
        x = self.tok(idx) + self.pos[:s]
        for blk in self.blocks:
            h = blk["ln1"](x)
            q, k, v = blk["qkv"](h).view(b, s, 3, self.heads, -1).permute(2, 0, 3, 1, 4)
            att = (q @ k.transpose(-1, -2)) / (q.shape[-1] ** 0.5) + self.mask[:s, :s]
            y = (att.softmax(-1) @ v).transpose(1, 2).reshape(b, s, -1)
            x = x + blk["proj"](y)
            x = x + blk["out"](torch.nn.functional.gelu(blk["fc"](blk["ln2"](x))))
        return self.head(self.ln(x))


def lm_loss(module: nn.Module, batch) -> torch.Tensor:
    x, y = batch
    logits = module(x)
    return torch.nn.functional.cross_entropy(logits.reshape(-1, logits.shape[-1]), y.reshape(-1))


def synthetic_lm_batch(seed: int, micro: int = 4, seq: int = 64, vocab: int = 256,
                       device="cuda:0") -> Callable:
    """batch_fn(t, m): tokens of step t's microbatch m, a pure function of
    (seed, t, m) — canonical data addressing.  A fixed random bigram table
    makes the data learnable."""
    g = torch.Generator().manual_seed(seed)
    table = torch.randint(0, vocab, (vocab,), generator=g)

    def batch(t: int, m: int):
        gen = torch.Generator().manual_seed((seed * 1_000_003 + t) * 1_000_003 + m)
        start = torch.randint(0, vocab, (micro, 1), generator=gen)
        noise = torch.rand(micro, seq, generator=gen) < 0.1
        toks = [start[:, 0]]
        for i in range(seq):
            nxt = table[toks[-1]]
            rnd = torch.randint(0, vocab, (micro,), generator=gen)
            toks.append(torch.where(noise[:, i], rnd, nxt))
        seqs = torch.stack(toks, 1)
        return seqs[:, :-1].to(device), seqs[:, 1:].to(device)
    return batch
