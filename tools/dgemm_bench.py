"""TF/s of the batched FP64 DMMA GEMM (ldgmg_dgemm_nt_batched) on the SAI
QR's four products at the C5 level-0 shapes, for every tile variant
(LDGMG_DGEMM_VARIANT, read once per process -> one subprocess each).

  python tools/dgemm_bench.py            # all variants
  python tools/dgemm_bench.py --variant 2
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, M, N, K, alpha, beta, batch): m = 2808 rows, the first wide panel of
# a 2808 x 756 problem (692 trailing columns + 108 right-hand sides)
SHAPES = [("Y=V^T C", 64, 800, 2808, 1.0, 0.0, 200), ("Gram", 64, 64, 2808, 1.0, 0.0, 200),
          ("Z=T^T Y", 64, 800, 64, 1.0, 0.0, 200), ("C-=V Z", 2808, 800, 64, -1.0, 1.0, 200)]


def child(variant):
    sys.path.insert(0, ROOT)
    import torch
    import paper_2412_12506_b200 as g
    from paper_2412_12506_b200 import _lib as L
    ctx = g.Context(0)
    out = {"variant": variant}
    for name, M, N, K, alpha, beta, batch in SHAPES:
        lda, ldb, ldd = K, K, M
        A = torch.rand(batch * M * lda, dtype=torch.float64, device="cuda")
        B = torch.rand(batch * N * ldb, dtype=torch.float64, device="cuda")
        D = torch.rand(batch * N * ldd, dtype=torch.float64, device="cuda")

        def run():
            L.check(L.lib.ldgmg_dgemm_nt_batched(ctx.h, M, N, K, alpha, A.data_ptr(), lda, M * lda, B.data_ptr(),
                                                 ldb, N * ldb, beta, D.data_ptr(), ldd, N * ldd, batch))
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record()
        for _ in range(reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3 / reps
        out[name] = round(2.0 * M * N * K * batch / t / 1e12, 2)
        del A, B, D
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variant", type=int, default=None)
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.child:
        child(a.variant)
        return
    for v in ([a.variant] if a.variant is not None else [0, 1, 2, 3, 4, 5]):
        env = dict(os.environ, LDGMG_DGEMM_VARIANT=str(v))
        r = subprocess.run([sys.executable, __file__, "--child", "--variant", str(v)], env=env, capture_output=True,
                           text=True, timeout=600)
        print(r.stdout.strip() or r.stderr[-2000:], flush=True)


if __name__ == "__main__":
    main()
