# interleaved A/B of larger first-load staggers (FB_FFT_STAGGER ns per CTA slot), 2048^2 and 1024^2 / 4096^2
cd $GRAFT_REPO_ROOT
rm -f gpurun_out/stagger2.jsonl
for r in 1 2 3; do
for cfg in "FB_FFT_STAGGER=300" "FB_FFT_STAGGER=600" "FB_FFT_STAGGER=900" "FB_FFT_STAGGER=1200"; do
for n in 2048 1024 4096; do
env $cfg timeout 60 python tools/fft_pass_bench.py $n $n 200 | sed "s/}}/, \"cfg\": \"$cfg\"}}/; s/{, /{/" >> gpurun_out/stagger2.jsonl 2>&1
done; done; done
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/stagger2.jsonl"):
    try:
        j = json.loads(l)
    except Exception:
        print(l.strip()); continue
    d[(j["n0"], j["knobs"].get("cfg", ""))].append(j["ms"] * 1e3)
for k, v in sorted(d.items()):
    print(f"{k[0]:6d} {k[1]:22s} " + " ".join(f"{x:.2f}" for x in v) + f"  mean {sum(v)/len(v):.2f} us")
PY
