"""Launch selected hot kernels a few times for ncu captures (run under gpurun + ncu).

    python scripts/profile_kernels.py euclid8192 [block]
    python scripts/profile_kernels.py suite8192          # every suite kernel, blocks 128/256/512/1024
    python scripts/profile_kernels.py reduce [n_rows]    # uniform 32-row table (configs[4] layout)
    python scripts/profile_kernels.py gemm8192 [block]
    python scripts/profile_kernels.py kernel NAME N BLOCK   # any suite kernel
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2103_14409_b200 as L  # noqa: E402


def main():
    what = sys.argv[1]
    c = L.Ctx(0)
    if what == "euclid8192":
        b = int(sys.argv[2]) if len(sys.argv) > 2 else 512
        reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
        c.register_suite([L.K_EUCLID], [8192])
        for _ in range(reps):
            c.launch(L.K_EUCLID, 8192, b)
    elif what == "suite8192":
        ks = [L.K_EUCLID, L.K_MATVEC, L.K_ROWSUM, L.K_COLSUM, L.K_TRANSPOSE, L.K_AXPY,
              L.K_STENCIL5]
        c.register_suite(ks, [8192])
        for k in ks:
            for b in (128, 256, 512, 1024):
                for _ in range(2):
                    c.launch(k, 8192, b)
    elif what == "gemm8192":
        b = int(sys.argv[2]) if len(sys.argv) > 2 else 256
        c.register_suite([L.K_GEMM_BF16], [8192])
        for _ in range(3):
            c.launch(L.K_GEMM_BF16, 8192, b)
    elif what == "kernel":                 # kernel NAME N BLOCK
        k, n, b = L.KERNELS[sys.argv[2]], int(sys.argv[3]), int(sys.argv[4])
        c.register_suite([k], [n])
        for _ in range(3):
            c.launch(k, n, b)
    elif what == "reduce":
        n = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000_000
        t = c.gen_table(n, n // 256, preset=L.PRESET_T4, seed=1, offsets=False)
        o = L.reduce_opts(32, 8)
        for _ in range(3):
            c.reduce_table(t, o, per_group=False)
            c.stats(o, percentiles=[0.01, 0.5, 0.99])
    torch.cuda.synchronize()
    print("done", what, "launches", c.launch_count())


if __name__ == "__main__":
    main()
