cat > /tmp/vb.py <<'PY'
import json, sys, torch, bench, gen
import paper_2605_00342_b200 as ev
if len(sys.argv) > 1:
    ev.LIB_PATH = ev.LIB_PATH.replace("libevict.so", sys.argv[1])
r = bench.verify_bench(ev, gen, torch, torch.cuda.current_stream())
print(sys.argv[1:], {m: (round(r[m]["kernel_ms"], 4), round(r[m]["roofline"]["frac"], 3), round(r[m]["b64_cold_us"], 1)) for m in ("sample", "greedy")})
PY
for v in libevict_v4.so libevict_v8.so; do PYTHONPATH=$PWD timeout 300 python /tmp/vb.py $v 2>&1 | tail -1; done
