"""Small cases for compute-sanitizer (tools/sanitize.sh): every kernel family once.

tcgen05 attention (sparse with verticals, dense slash tiles, isolated-slash gather, DCA
pattern changes, dense tiles), the tcgen05 estimator + cluster selection (n >= 4096 uses
the 8-CTA cluster top-k), the CUDA-core paths, the recall check and the LSE merge."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_15383_b200 import device as D, synth  # noqa: E402


def main():
    dev = "cuda:0"
    for n, hq, hkv, chunk, budget, dca in [(1024, 4, 2, 256, (40, 120), (256, 640, 256)),
                                           (4608, 4, 1, 1536, (64, 700), (1536, 3072, 1536))]:
        q, k, v = synth.make_qkv(n, hq, hkv, kind="planted", seed=3, device=dev,
                                 rope_base=1e4)
        r = D.chunked_prefill(q, k, v, chunk_len=chunk, last_q=64, budget=budget,
                              position_mode="dca_continuous", dca=dca, kernel_path="tc",
                              return_recall=True, return_admitted=True)
        torch.cuda.synchronize()
        assert torch.isfinite(r["out"]).all()
        rd = D.chunked_prefill(q, k, v, chunk_len=chunk, last_q=64, budget=budget, mode="full",
                               position_mode="dca_continuous", dca=dca, kernel_path="tc")
        torch.cuda.synchronize()
        assert torch.isfinite(rd["out"]).all()
    # CUDA-core (fp32) path
    q, k, v = (x.float() for x in synth.make_qkv(512, 2, 1, kind="iid", seed=4, device=dev))
    r = D.chunked_prefill(q, k, v, chunk_len=256, last_q=64, budget=(16, 24),
                          position_mode="dca_continuous", dca=(128, 384, 128))
    torch.cuda.synchronize()
    print("sanitize cases ok")


if __name__ == "__main__":
    main()
