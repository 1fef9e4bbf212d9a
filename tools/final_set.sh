set -x
TAG=${TAG:-r02i}
mkdir -p gpurun_out/${TAG:-r02i}
python -m pytest tests -m gpu -q 2>&1 | tail -2 > gpurun_out/${TAG:-r02i}/gputest.txt
python bench.py > gpurun_out/${TAG:-r02i}/bench_c3.jsonl 2> gpurun_out/${TAG:-r02i}/bench_c3.err
python bench.py --config c4 --no-cpu-baseline > gpurun_out/${TAG:-r02i}/bench_c4.jsonl 2>/dev/null
for r in 0.1 0.5 1.0; do python bench.py --ratio $r --no-cpu-baseline --no-extras > gpurun_out/${TAG:-r02i}/bench_r$r.jsonl 2>/dev/null; done
python bench.py --config c5 --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/${TAG:-r02i}/bench_c5_n1.jsonl 2> gpurun_out/${TAG:-r02i}/bench_c5.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG:-r02i}/bench_reference_arm.jsonl 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG:-r02i}/launches.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${TAG:-r02i}/launches.csv > gpurun_out/${TAG:-r02i}/launches.txt
ncu --set full --import-source on --clock-control none -k regex:dbsa_attn_kernel -c 1 -o gpurun_out/${TAG:-r02i}/k3 python tools/kbench.py --stage 2 --batch 64 --reps 1 > /dev/null 2>&1
python tools/ncu_summary.py full gpurun_out/${TAG:-r02i}/k3.ncu-rep > gpurun_out/${TAG:-r02i}/k3_ncu_full.json
ncu --set full --import-source on --clock-control none -k regex:dbsa_attn_kernel -c 1 -o gpurun_out/${TAG:-r02i}/k1 python tools/kbench.py --stage 1 --reps 1 > /dev/null 2>&1
python tools/ncu_summary.py full gpurun_out/${TAG:-r02i}/k1.ncu-rep > gpurun_out/${TAG:-r02i}/k1_ncu_full.json
rm -f gpurun_out/${TAG:-r02i}/*.ncu-rep
cat gpurun_out/${TAG:-r02i}/gputest.txt; head -12 gpurun_out/${TAG:-r02i}/launches.txt
