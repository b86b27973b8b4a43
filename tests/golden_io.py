"""Loaders for the committed golden fixtures (tests/golden/*, made by make_golden.py)."""

import json
import os

import numpy as np

from paper_2605_26461_b200.world import entries_from_list, flat_from_dict

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_json(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def batches():
    for b in load_json("batches.json"):
        yield flat_from_dict(b["world"]), entries_from_list(b["entries"]), b["params"], b["expect"]


def truth_table():
    for r in load_json("truth_table.json"):
        yield r, flat_from_dict(r["world"]), entries_from_list(r["entries"])


def classify_c1():
    z = np.load(os.path.join(GOLDEN, "classify_c1.npz"))
    return {k: z[k] for k in z.files}


def as_tuples(d):
    """JSON turns tuples into lists; normalise the observables dict back."""
    return dict(labels=list(d["labels"]), isolation=[tuple(x) for x in d["isolation"]],
                benign=[tuple(x) for x in d["benign"]], fatal_reports=d["fatal_reports"],
                clients={k: tuple(v) for k, v in d["clients"].items()},
                scenarios=list(d["scenarios"]))
