"""Loaders for the autodiff fixtures (tests/golden/ad_*.json, made by
oracle/gen_autodiff_golden.py)."""
import json
import os

import numpy as np

from paper_1810_08061_b200 import ir
from paper_1810_08061_b200.values import TensorValue

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NAMES = ["ad_lstm_4x3", "ad_lstm_6x4", "ad_maml_h8", "ad_rnn_full", "ad_rnn_break"]


def load(name):
    with open(os.path.join(GOLDEN, name + ".json")) as f:
        d = json.load(f)
    d["graph_obj"] = ir.from_json(d["graph"])
    d["feed_values"] = {k: TensorValue(v["tensor"]["dtype"], tuple(v["tensor"]["shape"]),
                                       np.asarray(v["tensor"]["data"]))
                        for k, v in d["feeds"].items()}
    return d


def close(got, exp, tol):
    """max |a - b| / (1 + |b|) <= tol over flattened values"""
    a = np.asarray(got, dtype=np.float64).reshape(-1)
    b = np.asarray(exp, dtype=np.float64).reshape(-1)
    return a.shape == b.shape and float(np.max(np.abs(a - b) / (1 + np.abs(b)), initial=0.0)) <= tol
