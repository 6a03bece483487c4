"""Loader for the reference-generated fixtures in tests/golden/."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

LL_NAMES = ["ll_f32_n4", "ll_uneven", "ll_n1", "ll_fewer", "ll_bf16", "ll_f16",
            "ll_fp8s", "ll_fp8", "ll_dsv3_tiny", "ll_dsv3_bf16"]
HT_NAMES = ["ht_f32_2node", "ht_uneven", "ht_bf16", "ht_node8", "ht_4node", "ht_n1"]


def load(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    return {k: z[k] for k in z.files}


def ll_case(name):
    g = load(name)
    n, rpn, e, bmax, b, k, h, scales, seed = (int(x) for x in g["spec"])
    return dict(g=g, n=n, rpn=rpn, e=e, bmax=bmax, b=b, k=k, h=h, scales=bool(scales),
                seed=seed, dtype=str(g["dtype"]), stub=str(g["stub"]),
                tokens=[g[f"tokens{r}"] for r in range(n)],
                routing=[g[f"routing{r}"] for r in range(n)],
                weights=[g[f"weights{r}"] for r in range(n)])


def ht_case(name):
    g = load(name)
    n, rpn, e, b, k, h, seed = (int(x) for x in g["spec"])
    return dict(g=g, n=n, rpn=rpn, e=e, b=b, k=k, h=h, seed=seed, dtype=str(g["dtype"]),
                stub=str(g["stub"]),
                tokens=[g[f"tokens{r}"] for r in range(n)],
                routing=[g[f"routing{r}"] for r in range(n)],
                weights=[g[f"weights{r}"] for r in range(n)])
