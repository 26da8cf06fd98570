"""Print which shared-memory words one tcgen05 TF32 MMA reads for A(m, k)
under a few descriptor stride choices (layout discovery for MN-major operands)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2602_15883_b200 import _lib as X

    K = 8
    for a_mn, lbo, sbo in [(0, 2048, 128), (1, 128, 128), (1, 128, 512), (1, 512, 128), (1, 128, 2048), (1, 2048, 128)]:
        C = torch.zeros((128, 32), dtype=torch.float32, device="cuda")
        X.call("fr_debug_tc_raw", C.data_ptr(), K, a_mn, lbo, sbo, None)
        torch.cuda.synchronize()
        c = C.cpu().numpy()[:, :K].astype(int)
        print(f"a_mn={a_mn} lbo={lbo} sbo={sbo}")
        for m in (0, 1, 2, 3, 4, 5, 7, 8, 9, 31, 32, 64, 127):
            print(f"  m={m:3d}:", " ".join(f"{v:5d}" for v in c[m]))


if __name__ == "__main__":
    main()
