"""Parser for the hand-worked fixtures under tests/golden/ (test helper, no method arithmetic)."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    """Returns (input_image, [ (op, params: dict, payload_lines) ... ])."""
    blocks = []
    cur = None
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.rstrip("\n")
            if not line or (cur is None and line.startswith("#")):
                continue  # comments only before the first @block (image rows use '#')
            if line.startswith("@"):
                parts = line[1:].split()
                params = {}
                for p in parts[1:]:
                    k, v = p.split("=")
                    params[k] = int(v)
                cur = (parts[0], params, [])
                blocks.append(cur)
            else:
                cur[2].append(line)
    inp = image(blocks[0][2])
    return inp, blocks[1:]


def image(lines):
    return np.array([[1 if c == "#" else 0 for c in ln] for ln in lines], dtype=np.uint8)


def ints(lines):
    return np.array([[int(v) for v in ln.split()] for ln in lines], dtype=np.int64)


def events_of(img):
    ys, xs = np.nonzero(img)
    return (xs.astype(np.uint32) | (ys.astype(np.uint32) << 16)).astype(np.uint32)
