# the bench lines of the final state: stdout must be exactly one JSON line each
python bench.py > gpurun_out/s4_bench_final.json 2> gpurun_out/s4_bench_final.err
python bench.py --config c2 > gpurun_out/s4_bench_c2.json 2>/dev/null
python bench.py --config c2 --route bdbsc > gpurun_out/s4_bench_c2_bdbsc.json 2>/dev/null
python bench.py --config c1 --route bdbs > gpurun_out/s4_bench_c1.json 2>/dev/null
python bench.py --sharded --check --steps 5 > gpurun_out/s4_bench_sharded.json 2>/dev/null
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu > gpurun_out/s4_bench_torchrun1.json 2>/dev/null
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s4_bench_ref.json 2>/dev/null
python - <<EOF
import json
for f in ["final", "c2", "c2_bdbsc", "c1", "sharded", "torchrun1", "ref"]:
    txt = open("gpurun_out/s4_bench_%s.json" % f).read()
    lines = [l for l in txt.splitlines() if l.strip()]
    d = json.loads(lines[0])
    print(f, "lines", len(lines), "ms", round(d["ms_per_step"], 4), "profiled", d.get("profiled_ms_per_step"), "e2e", (d.get("e2e") or {}).get("ms_per_step"), "check", d.get("check"))
EOF
