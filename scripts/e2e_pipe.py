"""Host-state pipelined LSRK step on config 4: step time against the chunk
size, plus the device-only chunked sweep (no copies) and the plain stepper."""
import json, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__
__graft_entry__.build()
import bench
from paper_1608_03836_b200 import solver, _native

TRACE_ONLY = "--trace-only" in sys.argv
if TRACE_ONLY:
    sys.argv.remove("--trace-only")
mesh, cfg, medium, disc, desc = bench.build_problem("c4")
d = disc.dev
K, Np = d.K, disc.ref.Np
host = [torch.randn((K, Np), dtype=torch.float32).pin_memory() for _ in range(4)]
st = solver.FieldState.from_fields(host)
dt = 1e-5
ev = lambda: torch.cuda.Event(enable_timing=True)


def timed(fn, n=4):
    fn(); fn(); torch.cuda.synchronize()
    e0, e1 = ev(), ev()
    e0.record()
    for _ in range(n):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


if TRACE_ONLY:
    sys.argv = sys.argv[:1] + ["none"]
sp = solver.DeviceStepper(disc, fused=True)
hold = [disc.to_device(st)]
def dstep():
    hold[0] = sp.step(hold[0], dt)
print(json.dumps({"device_step_ms": timed(dstep)}), flush=True)
del hold, sp
sms = torch.cuda.get_device_properties(0).multi_processor_count
# raw PCIe copies of the whole state (pinned host <-> device), alone and both directions at once
dev = torch.empty((4, K, Np), dtype=torch.float32, device="cuda")
hout = torch.empty((4, K, Np), dtype=torch.float32).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def h2d():
    for f in range(4):
        dev[f].copy_(host[f], non_blocking=True)
def d2h():
    hout.copy_(dev, non_blocking=True)
def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        h2d()
    with torch.cuda.stream(s2):
        d2h()
    cur.wait_stream(s1); cur.wait_stream(s2)
nb = dev.numel() * 4
r = {"state_GB": nb / 1e9}
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = timed(fn)
    r[name + "_ms"] = ms
    r[name + "_GBs_per_dir"] = nb / (ms * 1e-3) / 1e9
print(json.dumps(r), flush=True)
del dev, hout
args = sys.argv[1:] or ["auto", str(3 * sms), str(2 * sms)]
for a in args:
    if a == "none":
        break
    if a == "auto":
        cb = None
    elif a.startswith("r"):      # ramped head: 1, 1, 1, 2 waves, then 3-wave chunks
        nblk = d.Kpad // d.fused
        head = [sms, sms, sms, 2 * sms]
        tail = [2 * sms, sms, sms, sms]
        mid = nblk - sum(head) - sum(tail)
        body = [3 * sms] * (mid // (3 * sms))
        if mid - sum(body):
            body.append(mid - sum(body))
        cb = head + body + tail
    elif a.startswith("w"):
        cb = solver.pipeline_chunks(d.Kpad // d.fused, sms, int(a[1:]))
    else:
        cb = int(a)
    pipe = solver.HostPipeline(disc, chunk_blocks=cb)
    r = {"chunk_blocks": a, "chunks": len(pipe.blocks), "span": int(max(pipe.hi - range(len(pipe.hi))))}
    r["e2e_ms"] = timed(lambda: pipe.step(st, dt))
    for la in (1, 2, 8, 64):
        pipe.lookahead = la
        r[f"e2e_ms_lookahead{la}"] = timed(lambda: pipe.step(st, dt))
    pipe.lookahead = 8
    # the same launch order without copies
    import ctypes
    s = ctypes.byref(d.struct)
    cur = lambda: ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    def sweep():
        for stg, c in pipe.schedule:
            b0, b1 = pipe.blocks[c]
            _native.call("wadg_stage_fused", s, ctypes.c_void_p(pipe.bufs[(stg - 1) % 2].data_ptr()),
                         ctypes.c_void_p(pipe.bufs[stg % 2].data_ptr()), ctypes.c_void_p(pipe.stepper.res.data_ptr()),
                         disc.flux.tau_p, disc.flux.tau_u, solver.LSRK4A[stg - 1], solver.LSRK4B[stg - 1], dt, b0, b1, cur())
    r["chunked_sweep_ms"] = timed(sweep)
    # the same sweep while unrelated H2D and D2H copies of the state run on two
    # other streams: how much do the copies slow the kernels down?
    big_d = torch.empty((4, K, Np), dtype=torch.float32, device="cuda")
    big_h = torch.empty((4, K, Np), dtype=torch.float32).pin_memory()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    def sweep_with_copies():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur); s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            for f in range(4):
                big_d[f].copy_(host[f], non_blocking=True)
        with torch.cuda.stream(s2):
            big_h.copy_(pipe.rows_out, non_blocking=True)
        sweep()
        cur.wait_stream(s1); cur.wait_stream(s2)
    r["chunked_sweep_with_concurrent_copies_ms"] = timed(sweep_with_copies)
    del big_d, big_h
    print(json.dumps(r), flush=True)
    del pipe
    torch.cuda.empty_cache()

# where the pipeline overhead goes: the same step with parts switched off
import ctypes
pipe = solver.HostPipeline(disc)
s = ctypes.byref(d.struct)
vp = lambda t: ctypes.c_void_p(t.data_ptr())
spp = lambda stm: ctypes.c_void_p(stm.cuda_stream)
out = torch.empty((4, K, Np), dtype=torch.float32, pin_memory=True)


def variant(copy_in=True, pack=True, copy_out=True, unpack=True, compute=True):
    cur = torch.cuda.current_stream()
    pipe.h2d.wait_stream(cur); pipe.d2h.wait_stream(cur)
    with torch.cuda.stream(pipe.h2d):
        for c, (k0, k1) in enumerate(pipe.elems):
            if copy_in:
                for f in range(4):
                    pipe.rows_in[f, k0:k1].copy_(host[f][k0:k1], non_blocking=True)
            if pack:
                _native.call("wadg_rows_to_fields", s, vp(pipe.rows_in), k0, k1, vp(pipe.bufs[0]), spp(pipe.h2d))
            pipe.ev_in[c].record(pipe.h2d)
    waited = -1
    for stg, c in pipe.schedule:
        if stg == 1 and pipe.hi[c] > waited:
            waited = int(pipe.hi[c]); cur.wait_event(pipe.ev_in[waited])
        b0, b1 = pipe.blocks[c]
        if compute:
            _native.call("wadg_stage_fused", s, vp(pipe.bufs[(stg - 1) % 2]), vp(pipe.bufs[stg % 2]),
                         vp(pipe.stepper.res), disc.flux.tau_p, disc.flux.tau_u, solver.LSRK4A[stg - 1],
                         solver.LSRK4B[stg - 1], dt, b0, b1, spp(cur))
        if stg == 5:
            pipe.ev_out[c].record(cur)
    with torch.cuda.stream(pipe.d2h):
        for c, (k0, k1) in enumerate(pipe.elems):
            pipe.d2h.wait_event(pipe.ev_out[c])
            if unpack:
                _native.call("wadg_fields_to_rows", s, vp(pipe.bufs[1]), k0, k1, vp(pipe.rows_out), spp(pipe.d2h))
            if copy_out:
                for f in range(4):
                    out[f, k0:k1].copy_(pipe.rows_out[f, k0:k1], non_blocking=True)
    cur.wait_stream(pipe.h2d); cur.wait_stream(pipe.d2h)


VARIANTS = (("all", {}), ("no_copies", dict(copy_in=False, copy_out=False)),
            ("no_pack_unpack", dict(pack=False, unpack=False)),
            ("no_copy_out", dict(copy_out=False, unpack=False)),
            ("no_copy_in", dict(copy_in=False, pack=False)),
            ("copies_only", dict(compute=False)))
for name, kw in ([] if TRACE_ONLY else VARIANTS):
    print(json.dumps({"variant": name, "ms": timed(lambda: variant(**kw))}), flush=True)


# per-launch timeline of one pipelined step (compute stream): idle gaps before launches
pipe = solver.HostPipeline(disc)
for _ in range(2):
    pipe.step(st, dt)
torch.cuda.synchronize()
start = torch.cuda.Event(enable_timing=True)
pipe.trace = []
start.record()
pipe.step(st, dt)
end = torch.cuda.Event(enable_timing=True)
end.record()
torch.cuda.synchronize()
tl = [(s_, c_, start.elapsed_time(a), start.elapsed_time(b)) for s_, c_, a, b in pipe.trace]
gaps, prev, busy = [], 0.0, 0.0
for s_, c_, a, b in tl:
    gaps.append((s_, c_, round(a - prev, 3)))
    busy += b - a
    prev = b
print(json.dumps({"step_ms": round(start.elapsed_time(end), 3), "first_start_ms": round(tl[0][2], 3),
                  "last_end_ms": round(tl[-1][3], 3), "kernel_busy_ms": round(busy, 3),
                  "idle_ms": round(sum(g[2] for g in gaps), 3), "n_launches": len(tl),
                  "largest_gaps (stage, chunk, ms)": sorted(gaps, key=lambda g: -g[2])[:12],
                  "stage1_launch_ends": [round(b, 2) for s_, c_, a, b in tl if s_ == 1]}), flush=True)
