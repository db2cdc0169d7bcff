"""Golden MNDL fixture written by the REFERENCE's own serializer
(convevo/model_io.py:48-68) for a small genome, plus the reference forward of
a fixed batch through it. Run in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_mndl.py
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("CONVEVO_SRC", "/root/reference/pkg/src"))
from convevo import genome as rgen  # noqa: E402
from convevo import model_io as rio  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
SMALL = ("id=small00000000000 parents= lr=0.003 momentum=0.9 batch_size=8 "
         "f0=conv:oc=8,k=3,s=1,relu=1 f1=pool:size=2,s=2 f2=conv:oc=16,k=3,s=2,relu=1 h0=dense:units=12")
SHAPE = (3, 20, 20)


def main():
    net = rgen.instantiate(rgen.parse_genome(SMALL), SHAPE, seed=0)
    path = os.path.join(OUT, "small.mndl")
    rio.save_network(net, path)
    x = np.random.default_rng(5).random((6, *SHAPE), dtype=np.float32)
    logits = net.forward(x)
    with open(os.path.join(OUT, "small_mndl.json"), "w") as fh:
        json.dump({"genome": SMALL, "input_shape": SHAPE, "batch_seed": 5, "batch": 6,
                   "logits": logits.astype(np.float64).tolist(), "bytes": os.path.getsize(path)}, fh)


if __name__ == "__main__":
    main()
