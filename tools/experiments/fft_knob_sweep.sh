# interleaved knob sweep of the 2048^2 forward FFT (fft_pass_bench: CUDA events, L2 flushed)
cd $GRAFT_REPO_ROOT
rm -f gpurun_out/knobs.jsonl
for r in 1 2 3; do
for cfg in "" "FB_FFT_STAGGER=0" "FB_FFT_STAGGER=150" "FB_FFT_STAGGER=600" "FB_FFT_COL_C=8" "FB_FFT_COL_C=2" "FB_FFT_ROW_NB=2" "FB_FFT_COL_NB=1" "FB_FFT_COL_NB=2" "FB_FFT_COLPAIR=1"; do
env $cfg timeout 60 python tools/fft_pass_bench.py 2048 2048 200 | sed "s/}}/, \"cfg\": \"$cfg\"}}/" >> gpurun_out/knobs.jsonl 2>&1
done; done
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/knobs.jsonl"):
    try:
        j = json.loads(l)
    except Exception:
        print(l.strip()); continue
    d[j["knobs"].get("cfg", "")].append(j["ms"] * 1e3)
for k, v in d.items():
    print(f"{k or 'default':24s} " + " ".join(f"{x:.2f}" for x in v) + f"  mean {sum(v)/len(v):.2f} us")
PY
