cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for v in default bulk0 default bulk0; do
  if [ "$v" = default ]; then timeout 900 python tools/shard_probe.py 1 2 4 8 >> gpurun_out/r3x_shard_$v.jsonl 2>> gpurun_out/r3x.err
  else STAMG_LIB=abl/$v.so timeout 900 python tools/shard_probe.py 1 2 4 8 >> gpurun_out/r3x_shard_$v.jsonl 2>> gpurun_out/r3x.err; fi
done
python - <<'PY'
import json
for v in ("default", "bulk0"):
    for line in open(f"gpurun_out/r3x_shard_{v}.jsonl"):
        line=line.strip()
        if line.startswith("{"):
            d=json.loads(line); print(v, json.dumps(d)[:700])
PY
