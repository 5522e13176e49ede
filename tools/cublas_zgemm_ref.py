"""cuBLAS complex128 GEMM throughput on the LU / solve update shapes (reference point for zgemm_sub_tma)."""
import torch


def bench(fn, flops, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps
    return t, flops / (t / 1e3) / 1e12


def main():
    dev = "cuda"
    n = 4096
    a = torch.randn(n, n, dtype=torch.complex128, device=dev)
    b = torch.randn(n, n, dtype=torch.complex128, device=dev)
    t, tf = bench(lambda: a @ b, 8.0 * n ** 3)
    print(f"cuBLAS zgemm {n}^3: {t:.2f} ms {tf:.2f} TF/s")
    for (bs, m, k, nn) in [(128, 4032, 64, 4032), (128, 3968, 128, 3968), (64, 4032, 64, 128), (64, 3968, 128, 128),
                           (16, 4032, 64, 4032), (16, 3968, 128, 3968), (16, 3840, 256, 3840)]:
        A = torch.randn(bs, m, k, dtype=torch.complex128, device=dev)
        B = torch.randn(bs, k, nn, dtype=torch.complex128, device=dev)
        C = torch.randn(bs, m, nn, dtype=torch.complex128, device=dev)
        t, tf = bench(lambda: C.baddbmm_(A, B, alpha=-1.0), 8.0 * bs * m * k * nn)
        print(f"cuBLAS batched zgemm C-=AB b={bs} {m}x{k}x{nn}: {t:.2f} ms {tf:.2f} TF/s")
    d = torch.randn(n, n, dtype=torch.float64, device=dev)
    t, tf = bench(lambda: d @ d, 2.0 * n ** 3)
    print(f"cuBLAS dgemm {n}^3: {t:.2f} ms {tf:.2f} TF/s")


if __name__ == "__main__":
    main()
