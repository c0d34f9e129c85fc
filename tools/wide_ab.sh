for w in 0 1 2 3; do RK_BP_WIDE_GROUPS=$w python tools/batch_probe.py par512 > gpurun_out/bw_par_$w.json 2>&1; RK_BP_WIDE_GROUPS=$w python tools/batch_probe.py fan512 > gpurun_out/bw_fan_$w.json 2>&1; done
python - <<'PY'
import json
for wl in ("par","fan"):
    for w in range(4):
        d=json.load(open(f"gpurun_out/bw_{wl}_{w}.json"))["by_batch"]
        print(wl, w, " ".join(f"b{b}:{d[b]['backproject_us_per_image']:.1f}" for b in ("4","8","12","16","32")))
PY
python -m pytest tests/test_projector_gpu.py -q -m gpu -k "wide or bitwise or single_lane" 2>&1 | tail -3
