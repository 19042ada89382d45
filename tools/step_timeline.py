"""Kernel timeline of one Varuna step (torch.profiler / CUPTI activity
records: name, stream, start, duration), GPT-2 at P=1, to see which kernels
overlap across streams (e.g. the dropout-mask kernel forked beside LN/QKV).

    python tools/step_timeline.py --m 32 --N 2 --dropout 0.1 --out gpurun_out/tl.json
"""
import argparse
import collections
import dataclasses
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_04007_b200 import ParallelConfig  # noqa: E402
from paper_2111_04007_b200.model import CONFIGS  # noqa: E402
from paper_2111_04007_b200.runtime import Varuna, synthetic_batch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="gpt2_355m")
ap.add_argument("--m", type=int, default=32)
ap.add_argument("--N", type=int, default=2)
ap.add_argument("--dropout", type=float, default=0.1)
ap.add_argument("--out", default="gpurun_out/step_timeline.json")
a = ap.parse_args()
cfg = dataclasses.replace(CONFIGS[a.config], dropout=a.dropout)
pc = ParallelConfig(1, 1, a.m, a.N, (0,) * cfg.n_layer)
v = Varuna(cfg, pc, seed=0, init_device="cuda")
b = {k: t.cuda() for k, t in synthetic_batch(cfg, a.m * a.N, 0).items()}
for _ in range(3):
    v.step(b)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    v.step(b)
    torch.cuda.synchronize()
ev = []
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() > 0:
        ev.append({"name": e.name, "stream": getattr(e, "device_resource_id", -1),
                   "start": e.time_range.start, "dur": e.time_range.elapsed_us()})
ev.sort(key=lambda x: x["start"])
t0 = ev[0]["start"] if ev else 0
for x in ev:
    x["start"] -= t0


def short(n):
    n = n.replace("(anonymous namespace)::", "").replace("void ", "")
    return n.split("<")[0].split("(")[0].split("::")[-1]


# per kernel family: total time, and the fraction of it overlapped by kernels on other streams
busy = collections.defaultdict(list)
for x in ev:
    busy[x["stream"]].append((x["start"], x["start"] + x["dur"]))
summary = collections.defaultdict(lambda: [0, 0.0, 0.0])
for x in ev:
    s, e = x["start"], x["start"] + x["dur"]
    ov = 0.0
    for st, iv in busy.items():
        if st == x["stream"]:
            continue
        for a0, a1 in iv:
            if a1 > s and a0 < e:
                ov += min(a1, e) - max(a0, s)
    k = short(x["name"])
    summary[k][0] += 1
    summary[k][1] += x["dur"]
    summary[k][2] += min(ov, x["dur"])
span = max(x["start"] + x["dur"] for x in ev) if ev else 0
rows = sorted(summary.items(), key=lambda kv: -kv[1][1])
with open(a.out, "w") as f:
    json.dump({"span_us": span, "streams": sorted(busy), "events": ev[:20000],
               "summary": {k: {"n": n, "us": round(t, 1), "overlapped_us": round(o, 1)}
                           for k, (n, t, o) in rows}}, f)
print(f"step span {span:.0f} us, {len(ev)} kernels on {len(busy)} streams")
print(f"{'kernel':40s} {'n':>5s} {'us':>10s} {'share':>6s} {'overlapped':>10s}")
for k, (n, t, o) in rows[:30]:
    print(f"{k[:40]:40s} {n:5d} {t:10.1f} {100 * t / span:5.1f}% {100 * o / max(t, 1e-9):9.1f}%")
