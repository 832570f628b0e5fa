import gzip
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def load_golden(name):
    with gzip.open(os.path.join(GOLDEN, name), "rt") as f:
        return [json.loads(line) for line in f if line.strip()]


@pytest.fixture(scope="session")
def walks():
    return {w["spec"]: w for w in load_golden("walks.jsonl.gz")}


@pytest.fixture(scope="session")
def flow_corpus():
    return load_golden("flow424242.jsonl.gz") + load_golden("flow7302.jsonl.gz")


@pytest.fixture(scope="session")
def slack_corpus():
    return load_golden("slack7102.jsonl.gz")
