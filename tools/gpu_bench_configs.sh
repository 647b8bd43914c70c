# gpurun session: bench lines of the secondary configs (one JSON per config under gpurun_out/).
#   gpurun --timeout 3600 -- 'bash tools/gpu_bench_configs.sh 3 4 ...'
mkdir -p gpurun_out
for c in "$@"; do
  case $c in
    1) args="--config 1 --steps 3000 --warmup 5";;  # >= 1 s timed region: the nvidia-smi clock sampler needs it
    3|5|5nw) args="--config $c --steps 2 --warmup 3";;
    *) args="--config $c --steps 1 --warmup 3";;
  esac
  echo "== config $c"
  timeout 2400 python bench.py $args > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
  echo "rc=$?"; python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/bench_c{c}.json").read().strip().splitlines()[-1])
except Exception as e:
    print("no json", e); sys.exit()
print({k: d.get(k) for k in ("value", "ms_per_step")}, "e2e", d["e2e"]["value"], "frac", d["roofline"]["frac"],
      "parity", d["parity"], "pre", d.get("preprocess_s"))
for b in d.get("buckets", []):
    print("  ", b)
PY
  tail -2 gpurun_out/bench_c$c.err
done
