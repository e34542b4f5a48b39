"""Markdown rows from bench_configs.py JSON lines (for BASELINE.md section 4.2).

    python tools/cfg_tables.py file.jsonl [...]"""
import json
import sys


def fmt(x, nd=1):
    return "—" if x is None else f"{x:,.{nd}f}".replace(",", " ")


for f in sys.argv[1:]:
    for line in open(f):
        d = json.loads(line)
        x = d.get("exchange_us") or {}
        lat = "—" if not x else f"{fmt(x.get('p50'))} / {fmt(x.get('p99'))} ({fmt(x.get('p50_transfer_only'))})"
        k = d.get("kernel_ms_per_rank")
        print(f"| {f.split('/')[-1]} | N={d['n_gpus']} | {d['engine']} {d['route']} | rate {d.get('rate_target_hz')} "
              f"-> {d['rate_hz']} Hz | **{fmt(d['steps_per_s'], 0)}** | {lat} | "
              f"{', '.join(f'{v:.2f}' for v in k) if k else '—'} | ids {fmt(d.get('ids_per_step'), 0)} | "
              f"{d['clocks']['sm_mhz']:.0f} MHz {','.join(d['clocks']['reasons'])} | part {d.get('partition')} |")
