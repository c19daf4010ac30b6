"""Fit the NVSwitch's multimem.ld_reduce...add(.acc::f32).bf16x2 result to candidate rounding
rules (reading Z23).  Input: the binary written by tools/nvls_round_probe.cu.

    python tools/nvls_round_fit.py gpurun_out/r02/nvls_round_D2.bin
"""
import json
import sys

import numpy as np


def bf16_to_f64(b):
    return (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def round_bf16(x, mode):
    """x: float64 array (exact values) -> bf16 bits under `mode`: rne, rna (half away), rz, ru/rd."""
    x = np.asarray(x, np.float64)
    out = np.zeros(x.shape, np.uint16)
    nz = x != 0
    a = np.abs(x[nz])
    e = np.floor(np.log2(a))
    e = np.maximum(e, -133.0)                      # subnormal grid of bf16 (min exp -126, 7 bits)
    ulp = np.exp2(e - 7)
    q = a / ulp                                     # in [128, 256)
    fl = np.floor(q)
    frac = q - fl
    if mode == "rne":
        up = (frac > 0.5) | ((frac == 0.5) & (fl % 2 == 1))
    elif mode == "rna":
        up = frac >= 0.5
    elif mode == "rz":
        up = np.zeros_like(frac, bool)
    elif mode == "raz":
        up = frac > 0
    else:
        raise ValueError(mode)
    m = (fl + up) * ulp
    v = np.where(x[nz] < 0, -m, m).astype(np.float32)
    out[nz] = (v.view(np.uint32) >> 16).astype(np.uint16)
    return out


def fp32_seq(vals):
    s = np.zeros(vals.shape[1], np.float32)
    for row in vals:
        s = (s + row.astype(np.float32)).astype(np.float32)
    return s.astype(np.float64)


def main(path):
    raw = open(path, "rb").read()
    D, N = np.frombuffer(raw[:8], np.int32)
    arr = np.frombuffer(raw[8:], np.uint16)
    ins = arr[:D * N].reshape(D, N)
    res = arr[D * N:].reshape(2, D, N)              # [acc32=1, acc32=0][issuer][N]
    vals = bf16_to_f64(ins)
    exact = vals.sum(axis=0)
    s32 = fp32_seq(vals)
    s32r = fp32_seq(vals[::-1])
    out = {"D": int(D), "N": int(N)}
    for ai, acc in enumerate(("acc_f32", "acc_bf16")):
        r = res[ai]
        out[acc] = {"issuers_agree": bool(all(np.array_equal(r[0], r[g]) for g in range(D)))}
        for name, ref in (("exact", exact), ("fp32_rank_order", s32), ("fp32_reverse", s32r)):
            for mode in ("rne", "rna", "rz", "raz"):
                exp = round_bf16(ref, mode)
                ok = exp == r[0]
                # -0 vs +0 are different bits; count them separately
                out[acc][f"{name}/{mode}"] = float(ok.mean())
        exp = round_bf16(exact, "rne")
        bad = np.nonzero(exp != r[0])[0][:12]
        out[acc]["examples_vs_exact_rne"] = [
            {"in": [float(v) for v in vals[:, i]], "exact": float(exact[i]),
             "got": float(bf16_to_f64(r[0][i:i + 1])[0]), "rne": float(bf16_to_f64(exp[i:i + 1])[0])} for i in bad]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
