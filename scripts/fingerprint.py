"""Print the input fingerprints (tests/problems.input_fingerprint) of configs generated on the host."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.problems import config_problem, input_fingerprint  # noqa: E402

for name in sys.argv[1:]:
    pb = config_problem(name, with_DL=False)
    print(json.dumps({name: {k: [float(a) for a in v] for k, v in input_fingerprint(pb).items()}}), flush=True)
