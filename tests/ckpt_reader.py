"""Independent numpy reader of the checkpoint file format documented in include/lamb.h."""
import numpy as np


def read_checkpoint(path):
    raw = open(path, "rb").read()
    assert raw[:8] == b"LAMBCKPT"
    version, world = np.frombuffer(raw[8:16], np.uint32)
    n_tensors, step, n_params, data_off = np.frombuffer(raw[16:48], np.int64)
    numel = np.frombuffer(raw[48:48 + 8 * n_tensors], np.int64)
    data = np.frombuffer(raw[data_off:data_off + 12 * n_params], np.float32).reshape(3, n_params)
    cum = np.concatenate([[0], np.cumsum(numel)])
    split = lambda a: [a[cum[i]:cum[i + 1]] for i in range(n_tensors)]
    return {"version": int(version), "world": int(world), "step": int(step), "numel": numel,
            "w": split(data[0]), "m": split(data[1]), "v": split(data[2])}
