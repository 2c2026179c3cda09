"""Oracle's own reader for the plan JSON (the plan is data shared with the CUDA path; the reader
is not).  Format: see workload/make_plans.py and include/tn.h."""
import json

import numpy as np


class Plan:
    def __init__(self, d):
        self.raw = d
        self.tensors = []
        for t in d["tensors"]:
            labels = list(t["labels"])
            data = np.asarray(t["data"], dtype=np.float64)
            z = data[0::2] + 1j * data[1::2]
            self.tensors.append((labels, z.reshape((2,) * len(labels)) if labels else z.reshape(())))
        self.open = list(d["open"])
        self.tree = [tuple(p) for p in d["tree"]]
        self.sliced = list(d.get("sliced", []))
        self.stem = list(d.get("stem", []))


def load(path_or_dict):
    if isinstance(path_or_dict, dict):
        return Plan(path_or_dict)
    with open(path_or_dict) as f:
        return Plan(json.load(f))
