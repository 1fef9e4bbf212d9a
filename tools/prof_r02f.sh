set -x
mkdir -p gpurun_out/r02f
# batch-1 K3 (packed split-KV schedule) and the narrow K5, one launch each under ncu --set full
ncu --set full --import-source on --clock-control none -k regex:dbsa_attn_kernel -c 1 -o gpurun_out/r02f/k3b1 python tools/kbench.py --stage 2 --batch 1 --reps 1 > gpurun_out/r02f/k3b1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:label_lse_kernel -c 1 -o gpurun_out/r02f/k5b1 python tools/k5bench.py --rows 13 --reps 1 > gpurun_out/r02f/k5b1.log 2>&1
python tools/ncu_summary.py full gpurun_out/r02f/k3b1.ncu-rep > gpurun_out/r02f/k3b1_ncu_full.json
python tools/ncu_summary.py full gpurun_out/r02f/k5b1.ncu-rep > gpurun_out/r02f/k5b1_ncu_full.json
# launch list of one batch-1 graph replay pass (stage 2, random pages)
REPS=2 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f/b1_launches.csv python tools/b1prof.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r02f/b1_launches.csv > gpurun_out/r02f/b1_launches.txt
python tools/b1gaps.py > gpurun_out/r02f/b1_timeline.txt 2>&1
cat gpurun_out/r02f/k3b1_ncu_full.json gpurun_out/r02f/k5b1_ncu_full.json; head -14 gpurun_out/r02f/b1_launches.txt
