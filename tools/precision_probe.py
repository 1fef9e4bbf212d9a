"""Label-score error of the stage-2 schedules vs the reference goldens (c1, g128, m64ex):
chunk-major with bf16 / fp32 partials and split-KV per query."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from test_gpu_pipeline import _encoded
from paper_2503_08640_b200 import engine, pipeline, tokenizer

for name in ("c1", "g128", "m64ex"):
    meta, a, w, task, mc, enc = _encoded(name)
    runner = pipeline.Runner(w, enc.cache, enc.index, task, mc)
    queries = meta["queries"]
    q_ids = [tokenizer.encode(task.template.render_query(q["query"])) for q in queries]
    ids = np.stack([a[f"q{qi}_units"] for qi in range(len(queries))]).astype(np.int64)
    ref = np.stack([a[f"q{qi}_label_scores"] for qi in range(len(queries))])
    sess = runner.session()
    for sched, dt in (("query", None), ("chunk", torch.float32), ("chunk", torch.bfloat16)):
        tabs, n_ctx = sess.chunks_for(ids)
        jobs = [engine.label_job(tabs[i], int(n_ctx[i]), q, sess.label_ids) for i, q in enumerate(q_ids)]
        plan = engine.Stage2Plan(sess.dm, jobs, schedule=sched)
        if dt is not None:
            plan.sched.part_o = plan.sched.part_o.to(dt)

        s, best = sess.run(jobs, plan)
        s = s.double().cpu().numpy()
        print(f"{name} {sched:5s} {str(dt):14s} max|d score| {np.abs(s - ref).max():.4f} mean {np.abs(s - ref).mean():.5f}")
