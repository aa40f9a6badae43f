SECONDS=0
python bench.py --gpus 2 --allow-shared > gpurun_out/bench_2rank_shared.json 2> gpurun_out/bench_2rank_shared.err
echo rc=$? wall=${SECONDS}s
python - <<PY
import json
d=json.loads([l for l in open("gpurun_out/bench_2rank_shared.json") if l.startswith("{")][-1])
print(d["n_gpus"], round(d["value"],2), round(d["e2e"]["value"],2), d["config"]["frames_per_gpu"], d.get("collectives"), d.get("cpu_affinity"), d.get("note"))
for w in d["workloads"]: print(w["workload"], round(w["value"],2), w["config"]["frames_per_gpu"], w["config"]["global_frames"], w["parity_vs_reference"]["mismatching_frames"])
PY
tail -3 gpurun_out/bench_2rank_shared.err
