"""Per-SM ceiling of the streaming kernels when their data is L2-resident.

Times back-to-back launches (no flush) of one windowed pass along axis 0 and of
BDBS (axis-0 pass + fused pair) on arrays of 16..64 MB (inside the 126 MB L2)
and on a 4 GiB array (HBM-bound), CUDA events around the whole loop.  Prints
algorithmic GB/s (2 N s per pass): if the L2-resident rate is far above the
HBM rate, the kernels are not SM-bound at HBM speed.
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
    st = torch.cuda.current_stream().cuda_stream
    for planes in (4, 8, 16, 1024):
        shape = (planes * 4, 1024, 1024) if planes < 1024 else (1024, 1024, 1024)
        shape = (planes, 1024, 1024)
        x = torch.rand(shape, device="cuda")
        out = torch.empty_like(x)
        N = x.numel()
        reps = 200 if planes < 1024 else 10
        for what in ("axis0", "axis1", "bdbs"):
            def run():
                if what == "bdbs":
                    ex.bdbs_included(ex.Tensor(ex.Float32AddOps(), x), (16, 16, 16))
                else:
                    _native.check(L.exsum_windowed_pass(x.data_ptr(), out.data_ptr(), 0, 0, 3,
                                                        _native.i64_array(shape),
                                                        0 if what == "axis0" else 1, 16, st))
            for _ in range(3):
                run()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                run()
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / reps
            passes = 2 if what == "bdbs" else 1
            gbs = 2 * passes * N * 4 / (ms / 1e3) / 1e9
            print(f"{what:6s} {shape} {N * 4 / 2**20:7.0f} MiB  {ms * 1e3:9.1f} us  {gbs:8.0f} GB/s "
                  f"({gbs / 148:.1f} GB/s per SM)", flush=True)
        del x, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
