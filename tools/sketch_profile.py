"""One KRP sketch contraction at the config-5b core shape (r=1000, n=128, l=320)
for ncu captures: a d=3 tensor whose middle core is 1000 x 128 x 1000, so the
second launch of the sketch kernel is exactly one 5b middle-mode step."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_03598_b200 as P  # noqa: E402


def main():
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = P.Context(0, stream.cuda_stream)
    r, n, ell = 1000, 128, 320
    t = P.TTTensor.random_philox([n, n, n], [1, r, r, 1], 5, ctx)
    for _ in range(int(os.environ.get("REPS", "2"))):
        P.krp_partial_contractions_rl(t, ell, seed=7)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
