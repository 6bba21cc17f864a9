"""World-size-2 data parallelism on CPU (gloo): the host side of the N>1 path.

Each rank derives the same global schedule ("deal" dispatch: W*A consecutive
batches of the shuffled per-replica plan, what Trainer::train_one does with
dispatch=deal), takes its own sub-batch, computes its gradient with the
reference oracle, and the gradients are summed with a gloo all-reduce, then
divided by the global token count (trainer.cpp:244, 264-265). The result must
equal the gradient of all the rows at once (the sum-then-divide contract that
makes W a pure throughput knob), and every rank must see the same schedule.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ARCH, V = "transformer_base_defaults", 1000
OV = {"max_tokens": 512, "seed": 1, "criterion": "label_smoothed_cross_entropy"}


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def deal_schedule(corpus, workers, accum, max_tokens, seed, step):
    import paper_1904_01038_b200 as sqf
    plan = sqf.make_batches(corpus, max_tokens, 0, seed)
    order = sqf.shuffle_epoch(len(plan), seed, 1)
    base = step * workers * accum
    return [[plan[order[base + w * accum + a]] for a in range(accum)] for w in range(workers)]


def worker(rank, world, port, out_path):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1904_01038_b200 as sqf
    from oracle import ref
    corpus = sqf.synthetic_corpus(200, V, V, 1.1, 1)
    sub = deal_schedule(corpus, world, 1, OV["max_tokens"], OV["seed"], 0)
    # every rank derives the same global schedule
    mine = torch.tensor([x for b in sub for m in b for x in m], dtype=torch.int64)
    gathered = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(gathered, mine)
    assert all(torch.equal(g, mine) for g in gathered)
    rt = ref.RefTrainer(ARCH, OV, corpus, V, V)
    g, st = rt.subbatch_grad(sub[rank][0])
    grad = torch.from_numpy(g.astype(np.float32))
    ntok = torch.tensor([float(st["ntokens"])])
    dist.all_reduce(grad)   # bucket order does not matter for a sum (trainer.cpp:75-87)
    dist.all_reduce(ntok)
    if rank == 0:
        np.save(out_path, (grad / ntok).numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gradient_sum_matches_single_replica(tmp_path):
    import sys
    sys.path.insert(0, ROOT)
    import paper_1904_01038_b200 as sqf
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle not built")
    out = str(tmp_path / "g.npy")
    mp.start_processes(worker, args=(2, free_port(), out), nprocs=2, join=True, start_method="spawn")
    dist_grad = np.load(out)
    corpus = sqf.synthetic_corpus(200, V, V, 1.1, 1)
    sub = deal_schedule(corpus, 2, 1, OV["max_tokens"], OV["seed"], 0)
    rt = ref.RefTrainer(ARCH, OV, corpus, V, V)
    g_all, st = rt.subbatch_grad(sub[0][0] + sub[1][0])
    want = g_all / st["ntokens"]
    err = np.abs(dist_grad - want) / np.maximum(1.0, np.abs(want))
    assert err.max() < 1e-5
    assert np.abs(want).max() > 0
