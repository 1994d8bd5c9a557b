"""Summarise a bench.py JSON line (per-T table, split, rooflines)."""
import json
import sys

line = [ln for ln in open(sys.argv[1]) if ln.startswith("{")][-1]
d = json.loads(line)
print(f"value {d['value']/1e6:.3f} M {d['unit']}  e2e {d['e2e']['value']/1e6:.3f} M  ms/step {d['ms_per_step']:.3f}"
      f"  split {d['split']['pm']}/{d['split']['dm']} r={d['split']['decode_steps_per_prefill_layer']:.2f}"
      f"  clocks {d['clocks']}")
print(f"ttft/tpot layer us {d['ttft_layer_us']:.0f}/{d['tpot_layer_us']:.0f}  time-sliced "
      f"{d['time_sliced']['tokens_per_s']/1e6:.3f} M {d['time_sliced']['ttft_layer_us']:.0f}/{d['time_sliced']['tpot_layer_us']:.0f}")
print("roofline", {k: d["roofline"][k] for k in ("achieved", "peak", "frac")}, "gemms", d["prefill_gemms"]["frac_of_partition_peak"])
print("decode attn", {k: v for k, v in d["roofline_decode_attn"].items() if k.startswith("sms")})
print("idle", {k: v for k, v in d["sm_idle_pct"].items() if k != "prefill_group_note"})
for e in d["per_T"]:
    s, c, t = e["split"], e["corun"], e["time_sliced"]
    rs = e.get("regret_sweep", {})
    print(f"T={e['T']:5d} {s['branch']:15s} {s['pm']}/{s['dm']} r={e['decode_steps_per_prefill_layer']:.2f} "
          f"co {c['tokens_per_s']/1e6:.3f}M {c['ttft_layer_us']:.0f}/{c['tpot_layer_us']:.0f}  "
          f"ts {t['tokens_per_s']/1e6:.3f}M {t['ttft_layer_us']:.0f}/{t['tpot_layer_us']:.0f}  "
          f"wins={e['corun_vs_time_sliced']['wins']} ratio={e['corun_vs_time_sliced']['tokens_per_s_ratio']:.3f} "
          f"chunked {[round(x['tokens_per_s']/1e6, 3) for x in e['chunked']]} "
          f"best {rs.get('best_measured', {}).get('dm')} regret {rs.get('estimator_regret')}")
    if "-v" in sys.argv:
        for cnd in rs.get("candidates", []):
            print("     ", cnd)
if d.get("cpu_baseline"):
    cb = dict(d["cpu_baseline"])
    print("cpu", json.dumps(cb)[:1500])
if d.get("roofline_targets_split"):
    print("hbm split", d["roofline_targets_split"])
