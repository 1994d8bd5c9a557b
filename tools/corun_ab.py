"""Co-run A/B between two builds of libb200hot.so: median prefill layer and
decode layer-step times of the config-2 co-run (Llama-3-8B, T prefill tokens
on pm SMs beside B=32 ctx-2048 decode on dm SMs), each library in its own
process, alternated A B A B A B.

    python tools/corun_ab.py LIB_A LIB_B [T pm dm]
"""
import json
import os
import statistics
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2504_19516_b200.device import lib

    lib.load(sys.argv[2])
    from paper_2504_19516_b200.device.corun import CoRunner
    from paper_2504_19516_b200.workload import MODEL_PRESETS

    T, pm, dm = (int(v) for v in sys.argv[3:6])
    cr = CoRunner(MODEL_PRESETS["llama3-8b"], T, 32, 2048)
    cr.corun(pm, dm, 3, 1.4)
    r = cr.corun(pm, dm, 12, 1.4)
    print(json.dumps({"prefill_us": 1e6 * statistics.median(r.prefill_layer_s),
                      "decode_us": 1e6 * statistics.median(r.decode_layer_s)}))
    sys.exit(0)

a, b = sys.argv[1], sys.argv[2]
args = sys.argv[3:6] or ["4096", "140", "8"]
res = {a: [], b: []}
for rep in range(3):
    for libp in (a, b):
        out = subprocess.run([sys.executable, __file__, "--child", libp, *args], capture_output=True, text=True)
        line = [x for x in out.stdout.splitlines() if x.startswith("{")]
        if not line:
            print(out.stderr[-2000:])
            sys.exit(1)
        res[libp].append(json.loads(line[-1]))
for libp in (a, b):
    print(json.dumps({"lib": libp, "prefill_us": statistics.median(x["prefill_us"] for x in res[libp]),
                      "decode_us": statistics.median(x["decode_us"] for x in res[libp]),
                      "runs": res[libp]}))
