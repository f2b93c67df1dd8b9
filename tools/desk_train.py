"""Desk-scale training runs (paper_2406_02052_b200/train.py): RevNet-18 on
the synthetic CIFAR-shaped grating task with the paper's recipe, backpropagation (J = 1)
against PETRA J = 4 for accumulation k in {1, 2, 4}; one GPU.  Prints one JSON object.
    python tools/desk_train.py [epochs] > profiles/r02/desk_train.json"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_02052_b200 import train as T  # noqa: E402


def main():
    epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    runs = []
    for J, k in ((1, 1), (4, 1), (4, 2), (4, 4)):
        t0 = time.time()
        r = T.train(J=J, k=k, epochs=epochs, log=lambda m: print(m, file=sys.stderr, flush=True))
        r["wall_s"] = round(time.time() - t0, 1)
        runs.append(r)
        print(f"J={J} k={k}: test accuracy {r['test_accuracy']:.4f}, test loss {r['test_loss']:.4f}",
              file=sys.stderr, flush=True)
    print(json.dumps({"task": "synthetic class-conditional Gaussians (SPEC.md:584), 3x32x32, 10 classes, smooth "
                              "templates 3 sigma apart, random crop + flip (no network for CIFAR-10)",
                      "recipe": "SGD Nesterov 0.9, wd 5e-4 (not on BN / biases), batch 64, lr 0.1*64k/256, "
                                "linear warm-up 5/300 of the run, x0.1 at 1/2 and 3/4 (PAPER.md:256)",
                      "runs": runs}))


if __name__ == "__main__":
    main()
