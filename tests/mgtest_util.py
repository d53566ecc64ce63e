"""Shared helpers for the test-suite (golden fixtures, cached generated problems)."""
import functools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


@functools.lru_cache(maxsize=None)
def golden():
    with open(os.path.join(ROOT, "tests", "golden", "spec_examples.json")) as f:
        return json.load(f)


@functools.lru_cache(maxsize=None)
def problem(name):
    from problems import configs
    return configs.build(name)
