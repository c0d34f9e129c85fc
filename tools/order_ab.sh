# A/B of the forward CTA launch order (RK_FWD_ORDER=0: planner order, 1: longest first)
for o in 0 1; do RK_FWD_ORDER=$o python tools/batch_probe.py par512 > gpurun_out/fo_par_$o.json 2>&1; RK_FWD_ORDER=$o python tools/batch_probe.py fan512 > gpurun_out/fo_fan_$o.json 2>&1; done
python - <<'PY'
import json
for wl in ("par","fan"):
    for o in range(2):
        d=json.load(open(f"gpurun_out/fo_{wl}_{o}.json"))["by_batch"]
        print(wl, o, " ".join(f"b{b}:{d[b]['forward_us_per_image']:.1f}" for b in ("1","2","4","8","16","32","64","128")))
PY
