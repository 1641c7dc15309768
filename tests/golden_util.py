"""Loader for tests/golden/hebatch_golden.json (produced from the unmodified reference by
tools/make_golden.py)."""
import json
import os

_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "hebatch_golden.json")


def load():
    with open(_PATH) as fh:
        return json.load(fh)


def ints(hex_list):
    return [int(h, 16) for h in hex_list]
