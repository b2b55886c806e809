"""Per-SM ceiling of the streaming kernels when their data is L2-resident.

Round-2 version: in + out of every L2 case together stay under ~80 MB of the
126 MB L2 (the first version used 64 MiB in + 64 MiB out, which does not fit).
For each shape it times back-to-back launches (no flush; CUDA events around
the loop, and CUDA-graph replay of the same loop to take launch gaps out) of

  * copy   -- torch's device-to-device copy of the array (the L2 / HBM
              bandwidth a plain streaming kernel reaches),
  * axis0  -- one windowed pass along axis 0 (k_axis_stream),
  * axis1  -- one windowed pass along axis 1 (k_axis_stream),
  * bdbs   -- axis-0 pass + fused pair (2 passes),

and prints algorithmic GB/s (2 N s per pass).  If the L2 rate of the passes is
far above their HBM rate, the kernels are not SM-bound at HBM speed and a
schedule that keeps the axis-0 intermediate in L2 can pay.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2106_00124_b200 as ex
    from paper_2106_00124_b200 import _native

    L = _native.load()
    s = torch.cuda.Stream()
    shapes = [(64, 64, 1024), (64, 160, 1024), (1024, 1024, 1024)]
    for shape in shapes:
        x = torch.rand(shape, device="cuda")
        out = torch.empty_like(x)
        N = x.numel()
        big = N * 4 > 2**30
        reps = 10 if big else 200
        for what in ("copy", "axis0", "axis1", "bdbs"):
            st = s.cuda_stream

            def run():
                if what == "copy":
                    out.copy_(x)
                elif what == "bdbs":
                    ex.bdbs_included(ex.Tensor(ex.Float32AddOps(), x), (16, 16, 16))
                else:
                    _native.check(L.exsum_windowed_pass(x.data_ptr(), out.data_ptr(), 0, 0, 3,
                                                        _native.i64_array(shape),
                                                        0 if what == "axis0" else 1, 16, st))
            with torch.cuda.stream(s):
                for _ in range(3):
                    run()
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                for _ in range(reps):
                    run()
                b.record(s)
                torch.cuda.synchronize()
                ms = a.elapsed_time(b) / reps
                gms = None
                if what != "bdbs":  # bdbs allocates its workspace per call
                    try:
                        g = torch.cuda.CUDAGraph()
                        with torch.cuda.graph(g, stream=s):
                            for _ in range(20):
                                run()
                        g.replay()
                        torch.cuda.synchronize()
                        a.record(s)
                        for _ in range(max(1, reps // 20)):
                            g.replay()
                        b.record(s)
                        torch.cuda.synchronize()
                        gms = a.elapsed_time(b) / (max(1, reps // 20) * 20)
                    except Exception as e:  # pragma: no cover
                        print("graph failed:", e)
            passes = 2 if what == "bdbs" else 1
            gbs = 2 * passes * N * 4 / (ms / 1e3) / 1e9
            line = (f"{what:6s} {str(shape):18s} {N * 4 / 2**20:6.0f} MiB in  "
                    f"{ms * 1e3:9.2f} us  {gbs:7.0f} GB/s ({gbs / 148:5.1f}/SM)")
            if gms:
                gg = 2 * passes * N * 4 / (gms / 1e3) / 1e9
                line += f"  graph {gms * 1e3:9.2f} us {gg:7.0f} GB/s ({gg / 148:5.1f}/SM)"
            print(line, flush=True)
        del x, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
