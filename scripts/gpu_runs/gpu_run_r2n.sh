set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
s=$(date +%s); timeout 1800 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/n_bench.json 2> gpurun_out/n_bench.err; echo "bench rc=$? wall=$(( $(date +%s) - s ))s"; cat gpurun_out/n_bench.json
s=$(date +%s); timeout 1800 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/n_ref.json 2> gpurun_out/n_ref.err; echo "ref rc=$? wall=$(( $(date +%s) - s ))s"; cat gpurun_out/n_ref.json
timeout 900 python scripts/shard_projection.py 1 2 4 8 > gpurun_out/n_proj.jsonl 2> gpurun_out/n_proj.err; echo "proj rc=$?"; cat gpurun_out/n_proj.jsonl; tail -5 gpurun_out/n_proj.err
