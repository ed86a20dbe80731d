# Interleaved A/B of fb_fft2d timings between environment variants (knobs or FB_LIB builds):
#   bash tools/ab_env.sh "FB_FFT_SCHED=1|FB_FFT_SCHED=0" "2048 2048;1024 1024" ROUNDS
# one fresh process per point; summary per (size, variant) at the end
cd $GRAFT_REPO_ROOT
VARS=${1:-" "}; SIZES=${2:-"2048 2048"}; ROUNDS=${3:-3}
rm -f gpurun_out/ab_env.jsonl
IFS='|' read -ra VV <<< "$VARS"
IFS=';' read -ra SZ <<< "$SIZES"
for r in $(seq $ROUNDS); do
  for sz in "${SZ[@]}"; do
    for v in "${VV[@]}"; do
      env $v timeout 120 python tools/fft_pass_bench.py $sz 100 | VAR="$v" python -c "import json,os,sys; d=json.loads(sys.stdin.read()); d['variant']=os.environ['VAR']; print(json.dumps(d))" >> gpurun_out/ab_env.jsonl 2>&1
    done
  done
done
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for ln in open("gpurun_out/ab_env.jsonl"):
    try: j = json.loads(ln)
    except Exception: print(ln.strip()); continue
    d[(j["n0"], j["n1"], j["variant"])].append(j["ms"] * 1e3)
for k in sorted(d): print(k, " ".join(f"{v:.2f}" for v in d[k]), " mean %.2f us" % (sum(d[k]) / len(d[k])))
PY
