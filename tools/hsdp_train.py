#!/usr/bin/env python
"""BASELINE configs[3]: Llama-style 1B (1.236 B parameters) trained with HSDP
— FSDP2 2-way shard inside each replica, the fault-tolerant canonical commit
across replicas — on 4 GPUs (2 shards x 2 replicas; the config's 4 replicas
need 8 GPUs).  M = 32 microbatches of 2 x 2048 tokens per step (G = 16 per
replica), K = 20 buckets, bf16 compute and bf16 reduce-scatter, fp32 master
shards and fp32 K-ACC accumulation.  Trains --steps steps failure-free, then
again with replica 1 (both of its shard ranks) lost during_sync on bucket 7
of step --fail-step, and reports step times and whether the surviving
replica's parameters are bitwise the failure-free ones.

    python tools/hsdp_train.py --out gpurun_out/hsdp_configs3.json
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
sys.path.insert(0, os.path.join(ROOT, "tests"))

from mp_util import failed, spawn  # noqa: E402


def llama(a):
    from transformers import LlamaConfig, LlamaForCausalLM
    cfg = LlamaConfig(hidden_size=a.hidden, intermediate_size=a.ffn, num_hidden_layers=a.layers,
                      num_attention_heads=32, num_key_value_heads=8, vocab_size=128256,
                      max_position_embeddings=a.seq, tie_word_embeddings=True,
                      attn_implementation="eager")
    torch.manual_seed(0)
    return LlamaForCausalLM(cfg)


def worker(rank, world, a, fail):
    torch.use_deterministic_algorithms(True)
    from paper_2605_11215_b200.hsdp import HSDPTrainer

    def batch(t, m):
        g = torch.Generator(device="cuda").manual_seed((7 * 1_000_003 + t) * 1_000_003 + m)
        x = torch.randint(0, 32000, (a.micro, a.seq + 1), generator=g, device="cuda")
        return x[:, :-1], x[:, 1:]

    def loss_fn(model, b):
        x, y = b
        logits = model(input_ids=x).logits
        return torch.nn.functional.cross_entropy(logits.float().reshape(-1, logits.shape[-1]),
                                                 y.reshape(-1))

    tr = HSDPTrainer(lambda: llama(a), batch, loss_fn, shards=2, replicas=world // 2,
                     g_init=32 // (world // 2), k_buckets=20, lr=1e-3)

    class Kill:
        t = -1

        def fire(self, phase, bucket=None):
            if fail and self.t == a.fail_step and phase == "during_sync" and bucket == 7:
                return [1]
            return []

    kill = Kill()
    rows = []
    for t in range(a.steps):
        kill.t = t
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out, loss = tr.step(t, kill)
        torch.cuda.synchronize()
        rows.append({"step": t, "wall_ms": (time.perf_counter() - t0) * 1e3, "loss": loss,
                     "losses_by_m": {str(m): v for m, v in tr.last_losses.items()},
                     "contrib_total": out.contrib_total, "w_cur": out.w_cur,
                     "computed": sum(1 for s, _ in tr.computed if s == t)})
    import hashlib
    h = hashlib.sha256()
    for p in tr.params:
        h.update(p.to_local().detach().float().cpu().numpy().tobytes())
    return {"rows": rows, "params_hash": h.hexdigest(),
            "replica": tr.replica, "shard": tr.shard, "shard_numel": tr.numel,
            "alive": tr.replica in tr.engine.comm.members,
            "kacc_slots": tr.pool.allocated}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--fail-step", type=int, default=2)
    ap.add_argument("--micro", type=int, default=2)
    ap.add_argument("--seq", type=int, default=2048)
    ap.add_argument("--hidden", type=int, default=2048)
    ap.add_argument("--ffn", type=int, default=8192)
    ap.add_argument("--layers", type=int, default=16)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    world = 4
    ref = spawn(worker, world, a, False, timeout=3000)
    if failed(ref):
        print(json.dumps({"failed": failed(ref)}))
        sys.exit(1)
    got = spawn(worker, world, a, True, timeout=3000)
    if failed(got):
        print(json.dumps({"failed": failed(got)}))
        sys.exit(1)
    surv = [r for r in range(world) if got[r]["alive"]]

    def committed_losses(run):
        """Per step: the mean over all 32 committed microbatch losses, folded
        in microbatch-index order from whichever replica admitted each one
        (every shard rank of a replica reports the same values)."""
        out = []
        for t in range(a.steps):
            by_m = {}
            for r in range(world):
                by_m.update({int(m): v for m, v in run[r]["rows"][t]["losses_by_m"].items()})
            tot = 0.0
            for m in sorted(by_m):
                tot += by_m[m]
            out.append({"loss": tot / len(by_m), "microbatches": len(by_m)})
        return out
    loss_ref, loss_got = committed_losses(ref), committed_losses(got)
    same = all(got[r]["params_hash"] == ref[r]["params_hash"] for r in surv)
    steady = sorted(x["wall_ms"] for x in ref[0]["rows"][1:])
    doc = {
        "config": "configs[3]: Llama-style 1B HSDP, 2-way FSDP2 shard x 2 replicas on 4 GPUs",
        "params": 1_235_814_400 if (a.hidden, a.layers) == (2048, 16) else None,
        "shard_numel": ref[0]["shard_numel"], "microbatches": 32,
        "tokens_per_microbatch": a.micro * a.seq,
        "step_wall_ms_failure_free": [x["wall_ms"] for x in ref[0]["rows"]],
        "step_wall_ms_with_failure": [x["wall_ms"] for x in got[0]["rows"]],
        "failure": {"step": a.fail_step, "replica": 1, "during_sync_bucket": 7},
        "committed_tokens_per_s_failure_free": 32 * a.micro * a.seq / (steady[len(steady) // 2] / 1e3),
        "contrib_total": [x["contrib_total"] for x in got[0]["rows"]],
        "w_cur": [x["w_cur"] for x in got[0]["rows"]],
        "computed_by_replica0": [x["computed"] for x in got[0]["rows"]],
        "survivor_params_bitwise_equal_failure_free": same,
        "kacc_slots_per_rank": got[0]["kacc_slots"],
        "committed_loss_failure_free": [x["loss"] for x in loss_ref],
        "committed_loss_with_failure": [x["loss"] for x in loss_got],
        "committed_loss_microbatches": [x["microbatches"] for x in loss_got],
        "loss_trajectory_bitwise_equal": [x["loss"] for x in loss_ref] == [x["loss"] for x in loss_got],
        "losses_replica0_failure_free": [x["loss"] for x in ref[0]["rows"]],
        "losses_replica0_with_failure": [x["loss"] for x in got[0]["rows"]],
    }
    print(json.dumps(doc))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(doc, f, indent=1)
    sys.exit(0 if same else 2)


if __name__ == "__main__":
    main()
