"""Latency study: phase timestamps (%globaltimer) of the one-launch small-batch kernel.

`python tools/tiny_trace.py build` (here, CPU) compiles an instrumentation copy of the library
with -DCOSINE_TRACE into tools/_trace/pkg/ (the product build has no instrumentation);
`python tools/tiny_trace.py run [c1|c2]` (GPU) imports that copy, runs calls with L2 flushed
before each, and prints per phase the min / median / max over CTAs of the time since the
earliest CTA start (µs).  Slots: 0 start, 1 stats done, 2 unit decided (deciding CTAs),
3 request's decisions seen (parts), 4 request loaded, 5 part's tile masses done, 6 crossing
tile found (last part), 7 part end; inside the decision (deciding CTAs): 8 start, 9 gathers and
records combined, 10 confidences, 11 fusion and q(x*), 12 Philox, 13 acceptance, 14 written.
"""
import ctypes
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VARIANT = os.environ.get("TRACE_VARIANT", "")  # "noncoop": the one-launch kernel without the cooperative attribute
TR = os.path.join(ROOT, "tools", "_trace" + VARIANT)
PKGDST = os.path.join(TR, "pkg", "paper_2503_10325_b200")


def build():
    sys.path.insert(0, os.path.join(ROOT, "paper_2503_10325_b200"))
    import build as B
    os.makedirs(os.path.join(TR, "obj"), exist_ok=True)
    os.makedirs(PKGDST, exist_ok=True)
    objs = []
    procs = []
    for src in B.SOURCES:
        o = os.path.join(TR, "obj", os.path.basename(src)[:-3] + ".o")
        objs.append(o)
        procs.append(subprocess.Popen([B.nvcc(), *B.NVCC_FLAGS, "-DCOSINE_TRACE", *(["-DCOSINE_TRACE_NONCOOP"] if VARIANT == "noncoop" else []), "-I", B.INCLUDE, "-I", B.CSRC,
                                       "-c", "-o", o, src], stdout=subprocess.PIPE, stderr=subprocess.PIPE))
    for p in procs:
        out, err = p.communicate()
        if p.returncode:
            sys.stderr.write(err.decode())
            raise SystemExit("nvcc failed")
    for f in os.listdir(os.path.join(ROOT, "paper_2503_10325_b200")):
        if f.endswith(".py"):
            shutil.copy(os.path.join(ROOT, "paper_2503_10325_b200", f), PKGDST)
    subprocess.check_call([B.nvcc(), *B.ARCH, "-shared", "-o", os.path.join(PKGDST, "libcosine_verify.so"),
                           *objs, "-lnccl"])
    print("built", PKGDST)


def run(cfg, flush=True):
    sys.path.insert(0, os.path.join(TR, "pkg"))
    sys.path.insert(1, ROOT)
    import numpy as np
    import torch
    import paper_2503_10325_b200 as cv
    import synth
    assert cv.__file__.startswith(TR), cv.__file__
    lib = ctypes.CDLL(os.path.join(PKGDST, "libcosine_verify.so"))
    lib.cosine_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    lib.cosine_trace_read.restype = ctypes.c_size_t
    c = synth.CONFIGS[cfg]
    inp = synth.linear_inputs(c["B"], c["k"], c["N"], c["V"], dtype=c["dtype"], seed=3, device="cuda")
    ver = cv.Verifier(c["V"], max_batch=c["B"], k=c["k"], N=c["N"], device=0, target_dtype=c["dtype"],
                      draft_dtype=c["dtype"], seed=1)
    scratch = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
    rows = []
    ev_us = []
    for it in range(12):
        if flush:
            scratch.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ver.verify(inp["target"], inp["draft"], inp["draft_tokens"], inp["request_ids"], temperature=1.0)
        e1.record()
        torch.cuda.synchronize()
        if it >= 2:
            ev_us.append(e0.elapsed_time(e1) * 1e3)
        grid = cv.cosine_last_launch_count(ver.ctx)
        buf = np.zeros(1 << 20, dtype=np.uint64)
        n = lib.cosine_trace_read(buf.ctypes.data, buf.size)
        t = buf[:n].reshape(-1, 16).astype(np.int64)
        if it >= 2:
            rows.append(t)
    print(f"{cfg} (L2 {'flushed' if flush else 'warm'}{', ' + VARIANT if VARIANT else ''}): {rows[0].shape[0]} CTAs, "
          f"last launch count {grid}, call (events) median {np.median(ev_us):.2f} us")
    for slot in range(16):
        vals = []
        for t in rows:
            t0 = t[:, 0][t[:, 0] > 0].min()
            v = t[:, slot][t[:, slot] > 0] - t0
            if v.size:
                vals.append((v.min(), np.median(v), v.max()))
        if vals:
            a = np.array(vals, dtype=np.float64).mean(0) / 1e3
            print(f"  slot {slot}: min {a[0]:7.2f}  median {a[1]:7.2f}  max {a[2]:7.2f} us")


def run_split(cfg, select=0):
    """c3-size split path: per-kernel phase timestamps relative to the first stats CTA."""
    sys.path.insert(0, os.path.join(TR, "pkg"))
    sys.path.insert(1, ROOT)
    import numpy as np
    import torch
    import paper_2503_10325_b200 as cv
    import synth
    lib = ctypes.CDLL(os.path.join(PKGDST, "libcosine_verify.so"))
    lib.cosine_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    lib.cosine_trace_read.restype = ctypes.c_size_t
    c = synth.CONFIGS[cfg]
    inp = synth.linear_inputs(c["B"], c["k"], c["N"], c["V"], dtype=c["dtype"], seed=3, device="cuda")
    ver = cv.Verifier(c["V"], max_batch=c["B"], k=c["k"], N=c["N"], device=0, target_dtype=c["dtype"],
                      draft_dtype=c["dtype"], seed=1)
    res = []
    for it in range(6):
        ver.verify(inp["target"], inp["draft"], inp["draft_tokens"], inp["request_ids"], temperature=1.0,
                   select_mode=select)
        torch.cuda.synchronize()
        buf = np.zeros(1 << 23, dtype=np.uint64)
        n = lib.cosine_trace_read(buf.ctypes.data, buf.size)
        n_st, n_de, n_rs = (int(x) for x in buf[:3])
        t = buf[16:16 + 16 * (n_st + n_de + n_rs)].reshape(-1, 16).astype(np.int64)
        if it >= 2:
            res.append((t[:n_st], t[n_st:n_st + n_de], t[n_st + n_de:]))
    names = {"stats": {0: "start", 1: "done"}, "decide": {0: "start", 1: "unit ready", 2: "decided"},
             "resample": {0: "start", 1: "decisions seen", 5: "tile masses", 6: "crossing (last)", 7: "end"}}
    print(f"{cfg} split path (select {select}): grids {n_st} / {n_de} / {n_rs} CTAs")
    for gi, gname in enumerate(["stats", "decide", "resample"]):
        for slot, sname in names[gname].items():
            vals = []
            for r in res:
                t0 = r[0][:, 0][r[0][:, 0] > 0].min()
                v = r[gi][:, slot][r[gi][:, slot] > 0] - t0
                if v.size:
                    vals.append(np.percentile(v, [0, 10, 50, 90, 100]))
            if vals:
                a = np.array(vals).mean(0) / 1e3
                print(f"  {gname:8s} {sname:15s} " + "  ".join(f"{x:7.1f}" for x in a) + "   (min p10 p50 p90 max, us)")


def run_walk(cfg="c4", lazy=False):
    """The tree walk: per request CTA, time in the walk logic and in each kind of block step."""
    sys.path.insert(0, os.path.join(TR, "pkg"))
    sys.path.insert(1, ROOT)
    import numpy as np
    import torch
    import paper_2503_10325_b200 as cv
    import synth
    lib = ctypes.CDLL(os.path.join(PKGDST, "libcosine_verify.so"))
    lib.cosine_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    lib.cosine_trace_read.restype = ctypes.c_size_t
    c = synth.CONFIGS[cfg]
    B, N, V, dt = c["B"], c["N"], c["V"], c["dtype"]
    t = synth.tree_inputs(B, N, V, dtype=dt, seed=3, device="cuda")
    nn = t["J"] + 1
    ctx = cv.cosine_verify_init(V, device=0, max_batch=B, max_draft_len=1, max_drafters=N, seed=1,
                                target_dtype=dt, draft_dtype=dt, max_tree_nodes=nn)
    al = torch.empty(B, dtype=torch.int32, device="cuda")
    an = torch.empty(B, nn, dtype=torch.int32, device="cuda")
    ot = torch.empty(B, nn, dtype=torch.int32, device="cuda")
    st = torch.empty(B, dtype=torch.int32, device="cuda")
    res = []
    for it in range(5):
        cv.cosine_verify_tree(ctx, t["parent"], t["node_token"], t["internal_row"], t["target"], t["draft"],
                              t["node_draft_tokens"], t["request_ids"], al, an, ot, st, temperature=1.0, lazy=lazy)
        torch.cuda.synchronize()
        buf = np.zeros(B * 16, dtype=np.uint64)
        lib.cosine_trace_read(buf.ctypes.data, buf.size)
        if it >= 2:
            res.append(buf.reshape(B, 16).astype(np.int64))
    r = res[-1]
    t0 = r[:, 0].min()
    span = (r[:, 1] - r[:, 0]) / 1e3
    names = ["logic", "pass", "final", "stats", "error"]
    print(f"{cfg} walk ({'lazy' if lazy else 'all nodes'}): {B} CTAs; start spread {(r[:, 0].max() - t0) / 1e3:.1f} us; "
          f"end max {(r[:, 1].max() - t0) / 1e3:.1f} us")
    print(f"  per CTA span: median {np.median(span):.1f} max {span.max():.1f} us")
    order = np.argsort(-span)
    for q, nm in enumerate(names):
        acc = r[:, 2 + q] / 1e3
        cnt = r[:, 7 + q]
        print(f"  {nm:6s}: median {np.median(acc):7.1f} us  (slowest CTA {acc[order[0]]:7.1f} us, "
              f"count median {np.median(cnt):.0f}, slowest {cnt[order[0]]})")


if __name__ == "__main__":
    if sys.argv[1] == "walk":
        run_walk(sys.argv[2] if len(sys.argv) > 2 else "c4", "lazy" in sys.argv)
        raise SystemExit
    if sys.argv[1] == "split":
        run_split(sys.argv[2] if len(sys.argv) > 2 else "c3", int(sys.argv[3]) if len(sys.argv) > 3 else 0)
        raise SystemExit
    if sys.argv[1] == "build":
        build()
    else:
        run(sys.argv[2] if len(sys.argv) > 2 else "c1", flush="noflush" not in sys.argv)
