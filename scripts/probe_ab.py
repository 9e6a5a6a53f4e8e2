"""A/B timing of librmpb builds (RMPB_LIBRARY) on the bench workload:
4096 poses x 65536 rays, C1 map, L2 flushed between reps; prints one line."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_08068_b200 import synth
from paper_2301_08068_b200.device import RayPolicyEngine
import paper_2301_08068_b200 as P

PB = int(os.environ.get("PROBE_P", "4096"))
from paper_2301_08068_b200 import _lib
if os.environ.get("SEG_RAYS"):
    _lib.call("rmpb_set_option", b"seg_rays", int(os.environ["SEG_RAYS"]))
if os.environ.get("KERNEL"):
    _lib.call("rmpb_set_option", b"kernel", int(os.environ["KERNEL"]))
if os.environ.get("CARVEOUT"):
    _lib.call("rmpb_set_option", b"carveout", int(os.environ["CARVEOUT"]))
if os.environ.get("TRACE_WARPS"):
    _lib.call("rmpb_set_option", b"trace_warps", int(os.environ["TRACE_WARPS"]))
if os.environ.get("L2_WINDOW"):
    _lib.call("rmpb_set_option", b"l2_window", int(os.environ["L2_WINDOW"]))
scene = synth.c1_scene(); grid = synth.c1_grid(scene)
states = synth.bench_states(scene, count=PB, seed=123)
x_h, v_h = synth.states_arrays(states)
bundle = P.sample_directions(65536)
MR = float(os.environ.get("MAX_RANGE", "10.0"))
gsrc = grid
if os.environ.get("LAYOUT"):  # e.g. 4 = PAIR64 (librmpb LAYOUT_*)
    from paper_2301_08068_b200._kernels import b200
    gsrc = b200.DeviceGrid(grid.values, grid.origin, grid.resolution,
                           storage=int(os.environ.get("STORAGE", "0")),
                           layout=int(os.environ["LAYOUT"]))
eng = RayPolicyEngine(gsrc, bundle, P.preset("static_map").obstacle.as_tuple(), MR)
x = torch.from_numpy(x_h).cuda(); v = torch.from_numpy(v_h).cuda()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
s0, a0 = eng.evaluate(x, v); torch.cuda.synchronize()
ts = []
for _ in range(int(os.environ.get("PROBE_REPS", "5"))):
    flush.zero_()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); s, a = eng.evaluate(x, v); e1.record(); e1.synchronize()
    ts.append(e0.elapsed_time(e1))
sl = s.cpu().numpy()
print(json.dumps({"lib": os.path.basename(os.environ.get("RMPB_LIBRARY", "") or "librmpb.so"),
                  "l2_window": os.environ.get("L2_WINDOW", "default"),
                  "seg_rays": os.environ.get("SEG_RAYS", "auto"),
                  "carveout": os.environ.get("CARVEOUT", "default"),
                  "trace_warps": os.environ.get("TRACE_WARPS", "8"), "max_range": MR, "layout": os.environ.get("LAYOUT", "auto"), "kernel": os.environ.get("KERNEL", "0"),
                  "ms_min": round(min(ts), 3), "ms_med": round(sorted(ts)[len(ts) // 2], 3),
                  "hits": int(sl[:, 12].sum()), "sum_a00": float(sl[:, 0].sum()),
                  "sum_b0": float(sl[:, 9].sum())}), flush=True)
