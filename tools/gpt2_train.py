#!/usr/bin/env python
"""GPT-2 124M trained data-parallel through the canonical executor on one
GPU, K-ACC accumulation, with a replica killed mid-step (BASELINE configs[1]
on one GPU: W = 8 replicas x G = 4 microbatches of 4 x 1024 tokens, K = 20
buckets, replica 3 killed during_sync on bucket 7 at step --fail-step).

It trains the same model twice from the same seed, failure-free and with
the failure, and reports per-step wall time, the loss trajectories (bitwise
equal is the north-star claim), the K-ACC memory against the O(log G)
bound, and the failure step's recovery split.

    python tools/gpt2_train.py --steps 6 --fail-step 3 --out gpurun_out/gpt2.json

Random-initialised weights (transformers GPT2LMHeadModel, eager attention,
bf16 autocast, deterministic algorithms) and synthetic token data that is a
pure function of (step, microbatch): no checkpoints or datasets needed.
"""

import argparse
import json
import os
import sys
import time

os.environ.setdefault("CUBLAS_WORKSPACE_CONFIG", ":4096:8")

import torch  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_11215_b200.executor import CanonicalExecutor  # noqa: E402


def gpt2(layers, d, heads, vocab=50257, ctx=1024):
    from transformers import GPT2Config, GPT2LMHeadModel
    cfg = GPT2Config(n_layer=layers, n_embd=d, n_head=heads, vocab_size=vocab,
                     n_positions=ctx, attn_implementation="eager",
                     resid_pdrop=0.0, embd_pdrop=0.0, attn_pdrop=0.0)
    return GPT2LMHeadModel(cfg)


def batches(seed, micro, seq, vocab, device, active=1024):
    """Tokens of step t's microbatch m: drawn from a fixed random
    sub-vocabulary of `active` ids with a generator seeded by (seed, t, m)."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    table = torch.randperm(vocab, generator=g)[:active].to(device)

    def batch(t, m):
        gen = torch.Generator(device=device).manual_seed((seed * 1_000_003 + t) * 1_000_003 + m)
        toks = table[torch.randint(0, active, (micro, seq + 1), generator=gen, device=device)]
        return toks[:, :-1], toks[:, 1:]
    return batch


def lm_loss(model, batch):
    x, y = batch
    with torch.autocast("cuda", dtype=torch.bfloat16):
        logits = model(input_ids=x).logits
    return torch.nn.functional.cross_entropy(logits.float().reshape(-1, logits.shape[-1]),
                                             y.reshape(-1))


class Kill:
    def __init__(self, step, bucket, victim):
        self.at = (step, bucket)
        self.victim = victim
        self.t = -1

    def fire(self, phase, bucket=None):
        if phase == "during_sync" and (self.t, bucket) == self.at:
            return [self.victim]
        return []


def run(args, fail):
    torch.manual_seed(args.seed)
    model = gpt2(args.layers, args.d, args.heads)
    ex = CanonicalExecutor(model, batches(args.seed, args.micro, args.seq, 50257, "cuda:0"),
                           lm_loss, args.w, args.g, args.k, lr=args.lr, kacc=not args.slots)
    kill = Kill(args.fail_step if fail else -1, args.bucket, args.victim)
    rows = []
    for t in range(args.steps):
        kill.t = t
        ex.engine.recovery_events = [] if fail and t == args.fail_step else None
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out, loss = ex.step(t, kill)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3
        row = {"step": t, "loss": loss, "loss_hex": float(loss).hex(), "wall_ms": ms,
               "contrib_total": out.contrib_total, "w_cur": out.w_cur,
               "recomputed": sum(1 for s, _, _ in ex.computed if s == t) - args.w * args.g}
        if out.events:
            row["events"] = out.events
            ev = ex.engine.recovery_events or []
            names = [n for n, _, _ in ev]
            if "fail" in names and "commit" in names:
                row["fail_to_commit_ms"] = ev[names.index("fail")][1].elapsed_time(
                    ev[len(names) - 1 - names[::-1].index("commit")][1])
            row["reform_host_ms"] = out.reform_host_s * 1e3
        rows.append(row)
        print(json.dumps(row), file=sys.stderr)
    params = ex.flat.clone()
    return rows, params, ex.memory_report()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=12)
    ap.add_argument("--d", type=int, default=768)
    ap.add_argument("--heads", type=int, default=12)
    ap.add_argument("--micro", type=int, default=4)
    ap.add_argument("--seq", type=int, default=1024)
    ap.add_argument("--w", type=int, default=8)
    ap.add_argument("--g", type=int, default=4)
    ap.add_argument("--k", type=int, default=20)
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--fail-step", type=int, default=3)
    ap.add_argument("--bucket", type=int, default=7)
    ap.add_argument("--victim", type=int, default=3)
    ap.add_argument("--lr", type=float, default=0.05)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--slots", action="store_true", help="per-microbatch slots instead of K-ACC")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    torch.use_deterministic_algorithms(True)
    ref_rows, ref_p, _ = run(args, fail=False)
    rows, p, mem = run(args, fail=True)
    steady = [r["wall_ms"] for r in ref_rows[1:]]
    doc = {
        "model": "gpt2-124m" if (args.layers, args.d) == (12, 768) else
        "gpt2 %d layers d=%d" % (args.layers, args.d),
        "params": int(ref_p.numel()), "replicas": args.w, "microbatches": args.w * args.g,
        "tokens_per_microbatch": args.micro * args.seq, "buckets": args.k,
        "accumulation": "slots" if args.slots else "K-ACC",
        "failure": {"step": args.fail_step, "victim": args.victim,
                    "during_sync_bucket": args.bucket},
        "loss_failure_free": [r["loss"] for r in ref_rows],
        "loss_with_failure": [r["loss"] for r in rows],
        "loss_bitwise_equal": [r["loss_hex"] for r in ref_rows] == [r["loss_hex"] for r in rows],
        "params_bitwise_equal": bool(torch.equal(ref_p, p)),
        "step_wall_ms_failure_free_median": sorted(steady)[len(steady) // 2] if steady else None,
        "step_wall_ms_with_failure": [r["wall_ms"] for r in rows],
        "failure_step": rows[args.fail_step] if 0 <= args.fail_step < len(rows) else None,
        "committed_tokens_per_s": args.w * args.g * args.micro * args.seq * len(rows)
        / (sum(r["wall_ms"] for r in rows) / 1e3),
        "kacc_memory": mem,
        "gpu": torch.cuda.get_device_name(0),
    }
    print(json.dumps(doc))
    if args.out:
        os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
        with open(args.out, "w") as f:
            json.dump(doc, f, indent=1)
    sys.exit(0 if doc["loss_bitwise_equal"] and doc["params_bitwise_equal"] else 4)


if __name__ == "__main__":
    main()
