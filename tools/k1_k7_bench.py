"""HBM rooflines of the stencil (K1, global operator apply) and the GMRES
vector kernels (K7) at config-3 sizes (1241 x 441 grid, 64 RHS, raster
kappa^2), CUDA events, 20 repetitions after 3 warm-ups, inputs (>= 280 MB)
larger than L2.  Algorithmic bytes: K1 16 (read) + 16 (write)
+ 8 (raster kappa^2) per node and RHS; dot 32 per element (two reads); norm
16; axpy 48 (two reads, one write); axpy_dot 64 (three reads, y rewritten:
y -= a x_prev then vdot(x, y)); combine (k vectors, y += sum c x) 16 (k + 2).
usage: python tools/k1_k7_bench.py [config]  -> one JSON line"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2002_05327_b200 import configs
from paper_2002_05327_b200.krylov import _Vec


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps / 1e3


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    s = configs.spec(cfg)
    b = configs.build(s)
    gop = b["gop"]
    full = b["partition"].grid.full_window()
    counts = b["partition"].grid.counts
    R = s.nrhs
    n = int(torch.tensor(counts).prod())
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn((R, n), dtype=torch.complex128, device="cuda", generator=g)
    y = torch.randn((R, n), dtype=torch.complex128, device="cuda", generator=g)
    z = torch.randn((R, n), dtype=torch.complex128, device="cuda", generator=g)
    peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    vec = _Vec(n)
    out = torch.empty(R, dtype=torch.complex128, device="cuda")
    a = torch.full((R,), 0.5 + 0.25j, dtype=torch.complex128, device="cuda")
    xs = [torch.randn((R, n), dtype=torch.complex128, device="cuda", generator=g) for _ in range(8)]
    cc = torch.randn((8, R), dtype=torch.complex128, device="cuda", generator=g)
    k2b = 8 if gop.kappa2_kind == "full" else 0
    cases = {
        "stencil_apply": (lambda: gop.apply(x.reshape((R,) + counts), region=full), (32 + k2b) * n * R),
        "vec_dot": (lambda: vec.dot(x, y, out), 32 * n * R),
        "vec_norm": (lambda: vec.norm(x, out), 16 * n * R),
        "vec_axpy": (lambda: vec.axpy(a, -1.0, x, y), 48 * n * R),
        "vec_axpy_dot": (lambda: vec.axpy_dot(a, z, y, x, out), 64 * n * R),
        "vec_combine8": (lambda: vec.combine(xs, cc, y), 16 * 10 * n * R),
    }
    res = {}
    for k, (fn, nbytes) in cases.items():
        t = timed(fn)
        gbs = nbytes / t / 1e9
        res[k] = {"ms": t * 1e3, "achieved_gbs": gbs, "frac": gbs / peak, "bytes": nbytes}
    print(json.dumps({"config": s.name, "nodes": n, "nrhs": R, "peak_gbs": peak,
                      "peak_source": "MEASURED_PEAKS.json", "kernels": res}))


if __name__ == "__main__":
    main()
