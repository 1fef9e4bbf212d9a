"""Worker of tests/test_gpu_multiproc.py: one rank of a two-process run of
the sharded paths on cuda:0 (gloo rendezvous on 127.0.0.1).

  python tests/_mp_sharded_worker.py RANK WORLD PORT OUT_JSON
"""

import hashlib
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, str(HERE.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2503_08640_b200 as P  # noqa: E402
from paper_2503_08640_b200 import engine, parallel, pipeline, tokenizer  # noqa: E402
from test_gpu_pipeline import _setup  # noqa: E402


def main():
    rank, world, port, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4]
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    meta, a, w, task, mc = _setup("c1")
    dm = w.device()
    enc = P.encode_pool(w, task, mc)  # the partition, index and unit refs, exactly as encode_pool makes them
    rendered = [pipeline.render_block(task.template, task.pool, m) for m in enc.partition.blocks]
    blocks = [(ids, hashlib.sha256(t.encode()).digest(), sp) for t, ids, sp in rendered]
    comm = parallel.DistComm()
    caches, pairs, ranges = engine.encode_pool_sharded(dm, blocks, mc.pattern, comm)
    # pages of this rank's own groups vs the single-process cache
    worst = 0.0
    (r_local, cache), = caches.items()
    g0, g1 = ranges[r_local]
    for g in range(g0, g1):
        for layer in range(w.config.n_layers):
            k, v = cache.segment(layer, g)
            k0, v0 = enc.cache.segment(layer, g)
            worst = max(worst, float(np.abs(k - k0).max()), float(np.abs(v - v0).max()))
    total_pairs = sum(comm.all_gather_object([sum(pairs.values())]))
    queries = meta["queries"]
    runner = pipeline.Runner(w, enc.cache, enc.index, task, mc)
    units = [[enc.index.unit_refs[int(u)] for u in a[f"q{qi}_units"]] for qi in range(len(queries))]
    q_ids = [tokenizer.encode(task.template.render_query(q["query"])) for q in queries]
    sh = engine.ShardedStage2(dm, caches, comm, ranges, units, q_ids, runner.label_ids)
    scores, best = sh.scores()
    res = {"rank": rank, "pairs": int(total_pairs), "page_err": worst,
           "scores": scores.double().cpu().numpy().tolist(),
           "labels": [runner.labels[int(i)] for i in best.cpu().numpy()],
           "halo": len(parallel.halo_plan(mc.pattern, ranges, enc.cache.n_blocks))}
    Path(out).write_text(json.dumps(res))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
