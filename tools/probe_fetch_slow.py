import cProfile, io, pstats, sys, time, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
from paper_2602_09725_b200 import fetch as FE, codec
def wrap(mod, name):
    orig = getattr(mod, name)
    def w(*a, **k):
        pr = cProfile.Profile(); pr.enable(); t = time.perf_counter()
        try:
            return orig(*a, **k)
        finally:
            pr.disable(); dt = time.perf_counter() - t
            if dt > 0.04:
                s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(6)
                print(f"SLOW {name} {dt*1e3:.1f} ms\n" + "\n".join(s.getvalue().splitlines()[6:16]), file=sys.stderr)
    setattr(mod, name, w)
wrap(codec, "decode_batch"); wrap(FE, "restore_unit"); wrap(FE, "restore_units")
from paper_2602_09725_b200 import _lib as _L
_orig_call = _L.call
def timed_call(name, *a):
    t = time.perf_counter()
    try:
        return _orig_call(name, *a)
    finally:
        dt = time.perf_counter() - t
        if dt > 0.005:
            print(f"SLOW lib {name} {dt*1e3:.1f} ms", file=sys.stderr)
_L.call = timed_call
import torch
_orig_empty = torch.empty
def timed_empty(*a, **k):
    t = time.perf_counter()
    r = _orig_empty(*a, **k)
    dt = time.perf_counter() - t
    if dt > 0.01:
        print(f"SLOW torch.empty {dt*1e3:.1f} ms shape={a} kw={ {x: str(y) for x, y in k.items()} }", file=sys.stderr)
    return r
torch.empty = timed_empty
import bench_fetch_live
sys.argv = ["x", "--rates", os.environ.get("RATES", "100,100,100,100,100,100"), "--res", os.environ.get("RES", "R240")]
bench_fetch_live.main()
