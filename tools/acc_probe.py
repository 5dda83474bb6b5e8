"""Explore the tcgen05 kind::f16 (bf16 x bf16 -> fp32) accumulator's rounding on one B200:
alignment window, rounding mode, and the worst error on adversarial operands. Prints JSON lines.
Uses tests/cuda/libtcprobe.so (tc_bf16_acc)."""
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
from tc_acc import bf16_bits, bf16_val, run_acc  # noqa: E402

u = 2.0 ** -24


def window():
    # one step: product 1 plus fifteen products 2^-j; does each tiny product survive?
    out = {}
    for j in range(20, 34):
        A = np.zeros((128, 64), np.float32)
        B = np.zeros((32, 64), np.float32)
        A[:, 0] = 1.0
        B[:, 0] = 1.0
        A[:, 1:16] = 2.0 ** -j
        B[:, 1:16] = 1.0
        for c in range(32):  # column c keeps c+? tiny terms: zero out B beyond count
            B[c, 1 + min(c, 15):16] = 0.0
        D = run_acc(A, B)
        exact = A.astype(np.float64) @ B.T.astype(np.float64)
        out[j] = [float((D[0, c] - 1.0) / 2.0 ** -j) for c in range(0, 16)]
    return out


def next_step():
    # accumulator 1 after step 1, then step 2 (K 16..31) adds n tiny products
    out = {}
    for j in range(20, 30):
        A = np.zeros((128, 64), np.float32)
        B = np.zeros((32, 64), np.float32)
        A[:, 0] = 1.0
        B[:, 0] = 1.0
        A[:, 16:32] = 2.0 ** -j
        for c in range(32):
            B[c, 16:16 + min(c, 16)] = 1.0
        D = run_acc(A, B)
        out[j] = [float((D[0, c] - 1.0) / 2.0 ** -j) for c in range(0, 17)]
    return out


def rounding():
    # C = 1 (has_c), one product p: 1 + p rounded?
    res = {}
    for name, p in [("0.25ulp", 0.25), ("0.5ulp", 0.5), ("0.75ulp", 0.75), ("1.5ulp", 1.5), ("-0.25ulp", -0.25),
                    ("-0.75ulp", -0.75)]:
        A = np.zeros((128, 64), np.float32)
        B = np.zeros((32, 64), np.float32)
        A[:, 0] = p * 2.0 ** -23
        B[:, 0] = 1.0
        Cm = np.ones((128, 32), np.float32)
        D = run_acc(A, B, Cm)
        res[name] = float((D[0, 0] - 1.0) / 2.0 ** -23)
    return res


def adversarial(trials=20, K=512, seed=0):
    rng = np.random.default_rng(seed)
    worst = {}
    for fam in ("loguniform", "one_big", "big_first_step", "alternating_scale", "uniform"):
        wr = 0.0
        ws = 0.0
        for t in range(trials):
            if fam == "loguniform":
                A = 2.0 ** rng.uniform(-30, 0, (128, K))
                B = 2.0 ** rng.uniform(-30, 0, (32, K))
            elif fam == "uniform":
                A = rng.random((128, K)) + 0.5
                B = rng.random((32, K)) + 0.5
            elif fam == "one_big":
                A = 2.0 ** rng.uniform(-25, -22, (128, K))
                B = np.ones((32, K)) * (1 + rng.random((32, K)) * 0.99)
                A[:, rng.integers(0, K)] = 1.0
            elif fam == "big_first_step":
                A = 2.0 ** rng.uniform(-26, -21, (128, K))
                B = np.ones((32, K)) * (1 + rng.random((32, K)) * 0.99)
                A[:, :16] = 1.0 + rng.random((128, 16))
            else:
                s = np.where((np.arange(K) // 16) % 2 == 0, 1.0, 2.0 ** -12)
                A = (rng.random((128, K)) + 0.5) * s
                B = rng.random((32, K)) + 0.5
            A = bf16_val(A.astype(np.float32))
            B = bf16_val(B.astype(np.float32))
            D = run_acc(A, B).astype(np.float64)
            exact = A.astype(np.float64) @ B.T.astype(np.float64)
            mag = np.abs(A).astype(np.float64) @ np.abs(B).T.astype(np.float64)
            r = (np.abs(D - exact) / mag).max() / u
            wr = max(wr, r)
            ws = max(ws, r / (K / 16))
        worst[fam] = {"max_err_over_sum_u": wr, "per_mma_step_u": ws}
    return worst


if __name__ == "__main__":
    print(json.dumps({"window": window()}))
    print(json.dumps({"next_step": next_step()}))
    print(json.dumps({"rounding": rounding()}))
    for K in (64, 256, 512):
        print(json.dumps({"adversarial_K": K, "worst": adversarial(K=K)}))
