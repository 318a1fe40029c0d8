"""RHS-group concurrency probe: one plan over the whole batch vs G plans
over RHS groups issued on G torch streams (the paper's Remark 2 -- right-
hand sides pipelined through the sweeps).  usage: python tools/split_probe.py [config]"""
import sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_2002_05327_b200 import FactorizationCache, configs
from paper_2002_05327_b200 import _engine
from paper_2002_05327_b200.ddm import SweepPlan
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
s = configs.spec(cfg); b = configs.build(s); f = configs.sources(s, b["grid"])
part, ops = b["partition"], b["ops"]
R = f.shape[0]
cache = FactorizationCache()
cache.prepare([ops[i] for i in part.subdomains()])
fd = torch.from_numpy(f.reshape(R, -1)).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = {}
for G in (1, 2, 4):
    plans = [_engine.DevicePlan(part, ops, cache, SweepPlan.default(part.dim).directions, R // G, "diagonal",
                                pipelined=True) for _ in range(G)]
    streams = [torch.cuda.Stream() for _ in range(G)]
    chunks = [fd[g * (R // G):(g + 1) * (R // G)].contiguous() for g in range(G)]
    outs = [None] * G

    def run():
        main = torch.cuda.current_stream()
        for g in range(G):
            streams[g].wait_stream(main)
            with torch.cuda.stream(streams[g]):
                outs[g], _ = plans[g].apply(chunks[g])
        for g in range(G):
            main.wait_stream(streams[g])
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        flush.zero_()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); run(); e.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(e))
    u = torch.cat(outs, 0)
    if G == 1:
        ref = u.clone()
    err = float((u - ref).abs().max() / ref.abs().max())
    res[G] = (sum(ts) / len(ts), R / (sum(ts) / len(ts) / 1e3), err)
    print(G, "groups: ms %.3f  RHS/s %.1f  max rel diff vs 1 group %.2e" % res[G], flush=True)

if len(sys.argv) > 2 and sys.argv[2] == "device-only":
    sys.exit(0)
# host-buffer path (pinned f / u halves on G streams)
fh = torch.from_numpy(f.reshape(R, -1)).pin_memory()
uh = torch.empty_like(fh).pin_memory()
for G in (1, 2, 4):
    plans = [_engine.DevicePlan(part, ops, cache, SweepPlan.default(part.dim).directions, R // G, "diagonal",
                                pipelined=True) for _ in range(G)]
    streams = [torch.cuda.Stream() for _ in range(G)]
    lib, _ = _engine.context()

    def run_host():
        main = torch.cuda.current_stream()
        for g in range(G):
            streams[g].wait_stream(main)
            with torch.cuda.stream(streams[g]):
                lib_, ctx = _engine.context()
                sl = slice(g * (R // G), (g + 1) * (R // G))
                _engine.N.check(lib_.ds_ddm_apply_host(ctx, plans[g].handle, fh[sl].data_ptr(),
                                                       uh[sl].data_ptr(), R // G))
        for g in range(G):
            main.wait_stream(streams[g])
        torch.cuda.synchronize()
    for _ in range(3):
        run_host()
    t0 = time.perf_counter()
    for _ in range(10):
        run_host()
    dt = (time.perf_counter() - t0) / 10
    print(G, "groups host path: ms %.3f  RHS/s %.1f" % (dt * 1e3, R / dt), flush=True)
