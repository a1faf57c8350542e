"""compute-sanitizer target (tests/test_sanitizer_gpu.py): one small call of
every libgar kernel family -- coordinate kernels (TMA ring and direct loads,
fp32 and bf16), both Gram kernels (tf32 n <= 16, fp16 operands n > 16),
selection, combine, MDA, the world-1 peer exchange -- on C1-sized inputs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2010_05888_b200 as gar  # noqa: E402
import synth  # noqa: E402


def main():
    d = 20_011
    for n, f in ((11, 2), (31, 7), (40, 9)):
        X = synth.make_gradients(n, f, d, seed=n, device="cuda")
        Xb = synth.to_bf16(X)
        for rule in ("average", "median", "trimmed_mean", "krum", "multi_krum", "bulyan", "mean_around_median"):
            if rule == "bulyan" and n < 4 * f + 3:
                continue
            a = gar.init(rule, n, f)
            a.aggregate(X, d=d)
            a.aggregate(Xb, d=d)
        ws = torch.empty(gar.gar_workspace_bytes("krum", n, 0, d), dtype=torch.uint8, device="cuda")
        slots = torch.zeros(n * n, dtype=torch.float64, device="cuda")
        flags = torch.zeros(4, dtype=torch.int32, device="cuda")
        G = torch.empty((n, n), dtype=torch.float64, device="cuda")
        gar.gar_gram_exchange(X, G, ws, [slots.data_ptr()], [flags.data_ptr()], 0, 1, 1, d=d)
    gar.init("mda", 7, 2).aggregate(synth.make_gradients(7, 2, 3001, seed=3, device="cuda"), d=3001)
    torch.cuda.synchronize()
    print("sanitize target ok")


if __name__ == "__main__":
    main()
