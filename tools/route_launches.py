"""Per-launch device times of one route call (the library's CUDA-event profiler).

    python tools/route_launches.py --shape 256,256,256 --dtype int64 --monoid max-i64 --route box-complement --box 8,8,8
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="256,256,256")
    ap.add_argument("--box", default="8,8,8")
    ap.add_argument("--dtype", default="int64")
    ap.add_argument("--monoid", default="max-i64")
    ap.add_argument("--route", default="box-complement")
    args = ap.parse_args()
    import torch
    import paper_2106_00124_b200 as ex
    from paper_2106_00124_b200 import _native
    shape = tuple(int(v) for v in args.shape.split(","))
    box = tuple(int(v) for v in args.box.split(","))
    g = torch.Generator(device="cuda").manual_seed(0)
    if args.dtype == "int64":
        x = torch.randint(-2**20, 2**20, shape, generator=g, device="cuda")
    else:
        x = torch.rand(shape, generator=g, device="cuda",
                       dtype=torch.float32 if args.dtype == "float32" else torch.float64)
    ops = ex.Float32AddOps() if args.monoid == "add-f32" else ex.resolve_monoid(args.monoid)
    t = ex.Tensor(ops, x)
    fn = {"bdbs": ex.bdbs_included, "bdbsc": ex.bdbs_excluded,
          "box-complement": ex.box_complement_excluded, "sat": ex.sat_included}[args.route]
    for _ in range(3):
        fn(t, box)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    _native.profile_enable(True)
    a.record()
    fn(t, box)
    b.record()
    torch.cuda.synchronize()
    for name, by, ms in _native.profile_records():
        print(f"  {name:18s} {by / 1e6:9.2f} MB {ms * 1e3:8.1f} us {by / ms / 1e9 if ms else 0:8.1f} GB/s")
    print(f"step {a.elapsed_time(b) * 1e3:.1f} us")
    _native.profile_enable(False)


if __name__ == "__main__":
    main()
