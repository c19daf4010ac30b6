"""Independent numpy reader of the checkpoint file format documented in include/lamb.h (v2)."""
import numpy as np


def read_checkpoint(path):
    raw = open(path, "rb").read()
    assert raw[:8] == b"LAMBCKPT"
    version, world = np.frombuffer(raw[8:16], np.uint32)
    assert version == 2, version
    n_tensors, step, n_params, data_off = np.frombuffer(raw[16:48], np.int64)
    session, save_seq = np.frombuffer(raw[48:64], np.uint64)
    numel = np.frombuffer(raw[64:64 + 8 * n_tensors], np.int64)
    commit = np.frombuffer(raw[64 + 8 * n_tensors:64 + 8 * n_tensors + 64], np.uint64)
    assert np.all(commit[:world] != 0), "a saving rank never committed"
    data = np.frombuffer(raw[data_off:data_off + 12 * n_params], np.float32).reshape(3, n_params)
    cum = np.concatenate([[0], np.cumsum(numel)])
    split = lambda a: [a[cum[i]:cum[i + 1]] for i in range(n_tensors)]
    return {"version": int(version), "world": int(world), "step": int(step), "numel": numel,
            "save_seq": int(save_seq), "commit": commit[:world].copy(),
            "w": split(data[0]), "m": split(data[1]), "v": split(data[2])}
