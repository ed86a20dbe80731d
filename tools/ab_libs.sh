# A/B of FFT timings between libfb.so builds: bash tools/ab_libs.sh "libA.so libB.so" "2048 2048;1024 1024" ROUNDS
# (interleaved, each point a fresh process; one JSON line per run in gpurun_out/ab_libs.jsonl)
cd $GRAFT_REPO_ROOT
LIBS=${1:-"libfb.so"}; SIZES=${2:-"2048 2048"}; ROUNDS=${3:-3}
rm -f gpurun_out/ab_libs.jsonl
for r in $(seq $ROUNDS); do
  IFS=';' read -ra SZ <<< "$SIZES"
  for sz in "${SZ[@]}"; do
    for L in $LIBS; do
      FB_LIB=paper_2004_09883_b200/$L timeout 120 python tools/fft_pass_bench.py $sz 100 | sed "s/}}/}, \"lib\": \"$L\"}/" >> gpurun_out/ab_libs.jsonl 2>&1
    done
  done
done
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for ln in open("gpurun_out/ab_libs.jsonl"):
    try: j = json.loads(ln)
    except Exception: continue
    d[(j["n0"], j["n1"], j["lib"])].append(j["ms"] * 1e3)
for k in sorted(d): print(k, " ".join(f"{v:.2f}" for v in d[k]), " mean %.2f us" % (sum(d[k]) / len(d[k])))
PY
