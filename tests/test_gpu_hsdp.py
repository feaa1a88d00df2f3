"""HSDP with FSDP2: 2 shards x 2 replicas of a small Llama.
Inside a replica, FSDP2 shards the parameters and reduce-scatters every
microbatch's gradient in bf16 with FSDP's divide switched off; across
replicas the shard gradients are accumulated by K-ACC and committed by the
fault-tolerant canonical commit.  The committed shard gradient is bitwise
the oracle's canonical tree over the reduce-scattered leaves / B, and a
replica's death mid-step changes no parameter bit of the survivor."""

import os

import numpy as np
import pytest
import torch

from mp_util import failed, spawn

pytestmark = [pytest.mark.gpu]


def _model():
    from transformers import LlamaConfig, LlamaForCausalLM
    cfg = LlamaConfig(hidden_size=128, intermediate_size=256, num_hidden_layers=2,
                      num_attention_heads=4, num_key_value_heads=2, vocab_size=512,
                      max_position_embeddings=64, attn_implementation="eager")
    torch.manual_seed(0)
    return LlamaForCausalLM(cfg)


def _batch(t, m):
    g = torch.Generator(device="cuda").manual_seed(1000 * t + m)
    x = torch.randint(0, 512, (2, 33), generator=g, device="cuda")
    return x[:, :-1], x[:, 1:]


def _loss(model, batch):
    x, y = batch
    logits = model(input_ids=x).logits
    return torch.nn.functional.cross_entropy(logits.float().reshape(-1, logits.shape[-1]),
                                             y.reshape(-1))


class Kill:
    def __init__(self, plan):
        self.plan = dict(plan)
        self.t = -1

    def fire(self, phase, bucket=None):
        e = self.plan.get(self.t)
        if e and e[0] == phase and (phase != "during_sync" or e[1] == bucket):
            del self.plan[self.t]
            return e[2]
        return []


def _worker(rank, world, plan):
    os.environ.setdefault("CUBLAS_WORKSPACE_CONFIG", ":4096:8")
    torch.use_deterministic_algorithms(True)
    import torch.distributed as dist
    from oracle import fold
    from paper_2605_11215_b200.hsdp import HSDPTrainer
    tr = HSDPTrainer(_model, _batch, _loss, shards=2, replicas=2, g_init=4, k_buckets=3,
                     lr=0.1, barrier_timeout_s=60.0)
    tr.capture = {}
    kill = Kill({t: tuple(v) for t, v in plan.items()})
    out_rows = []
    oracle_ok = None
    for t in range(3):
        kill.t = t
        out, _ = tr.step(t, kill)
        torch.cuda.synchronize()
        if t == 0:
            got = [None] * 2
            dist.all_gather_object(got, {m: v.numpy() for m, v in tr.capture.items()},
                                   group=tr.rep_pg)
            leaves = {m: v for d in got for m, v in d.items()}
            want = fold.canonical_tree(leaves, tr.b) / np.float32(tr.b)
            oracle_ok = tr.grad.cpu().numpy().tobytes() == want.tobytes()
        tr.capture = {}
        alive = tr.replica in tr.engine.comm.members
        out_rows.append((out.contrib_total, out.w_cur, alive))
    params = [p.to_local().detach().cpu().numpy().tobytes() for p in tr.params]
    tr.engine.check_peers()
    return {"rows": out_rows, "oracle_ok": oracle_ok, "params": params,
            "replica": tr.replica, "shard": tr.shard}


def test_hsdp_fsdp2_bitwise_through_replica_death():
    if torch.cuda.device_count() < 4:
        pytest.skip("FSDP2's NCCL shard group needs 4 distinct GPUs")
    ref = spawn(_worker, 4, {})
    assert not failed(ref), failed(ref)
    got = spawn(_worker, 4, {1: ("during_sync", 1, [1])})
    assert not failed(got), failed(got)
    for r in range(4):
        assert ref[r]["oracle_ok"] and got[r]["oracle_ok"], r
        assert [row[0] for row in got[r]["rows"]] == [8, 8, 8]
    # the surviving replica's shards: every parameter bit as without the death
    for r in (0, 1):
        assert got[r]["replica"] == 0 and got[r]["rows"][-1][2]
        assert got[r]["params"] == ref[r]["params"], r
