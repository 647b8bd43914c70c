import json
import sys
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libmgk.so")


def load_golden(name):
    return json.loads((GOLDEN / name).read_text())


def graph_from_json(d, cls=None):
    """Golden graph dict -> our LabeledGraph (or a plain namespace)."""
    def lab(x):
        if x is None:
            return None
        if x["kind"] == "categorical":
            return np.asarray(x["data"], dtype=np.int64)
        return np.asarray(x["data"], dtype=np.float64).reshape(len(x["data"]), -1)

    from paper_1910_06310_b200.graphs import LabeledGraph

    return LabeledGraph(
        node_count=d["n"],
        edges_i=np.asarray(d["ei"], dtype=np.int64),
        edges_j=np.asarray(d["ej"], dtype=np.int64),
        weights=np.asarray(d["w"], dtype=np.float64),
        start_prob=np.asarray(d["p"], dtype=np.float64),
        stop_prob=np.asarray(d["q"], dtype=np.float64),
        node_labels=lab(d["node_labels"]),
        edge_labels=lab(d["edge_labels"]),
    )


@pytest.fixture(scope="session")
def golden_structure():
    return load_golden("structure.json")


@pytest.fixture(scope="session")
def golden_kernels():
    return load_golden("kernels.json")


@pytest.fixture(scope="session")
def golden_gram():
    return load_golden("gram.json")


@pytest.fixture(scope="session")
def golden_rng():
    return load_golden("rng.json")
