S=/usr/local/cuda/bin/compute-sanitizer
echo "## memcheck: schedules (packed split-KV with cta_works + PDL, chunk-major, padded) at hd 128 GQA-4, K5 narrow + wide, K4"
timeout 900 $S --tool memcheck python -m pytest tests/test_gpu_kernels.py -m gpu -q -k "schedules_vs_float64 and 128-8-2 or label_score and (1-64 or 13-4096 or 130) or topk" 2>&1 | grep -E "ERROR SUMMARY|passed|failed|Invalid|out of bounds|Address|Program hit" | head -20
echo "## memcheck: Runner.infer (packed split-KV, PDL, templates, padding) and the graph-replayed chunk-major path with the last-layer subset, c1"
timeout 900 $S --tool memcheck python -m pytest tests/test_gpu_pipeline.py -m gpu -q -k "runner_matches_reference and c1 and packed-bf16] or benchmarked_path and c1" 2>&1 | grep -E "ERROR SUMMARY|passed|failed|Invalid|out of bounds|Address|Program hit" | head -20
echo "## racecheck: split-KV packed and chunk-major schedules at hd 128"
timeout 900 $S --tool racecheck python -m pytest tests/test_gpu_kernels.py -m gpu -q -k "schedules_vs_float64 and 128-8-2 and (query or chunk])" 2>&1 | grep -E "RACECHECK SUMMARY|passed|failed|hazard" | head -10
echo "## racecheck: K5 narrow"
timeout 900 $S --tool racecheck python -m pytest tests/test_gpu_kernels.py -m gpu -q -k "label_score and 5-64" 2>&1 | grep -E "RACECHECK SUMMARY|passed|failed|hazard" | head -10
