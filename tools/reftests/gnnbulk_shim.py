"""`import gnnbulk` resolves to the B200 package, so the reference's own
test files run unmodified against it (tools/reftests/prepare.sh)."""
import sys

import paper_2311_02909_b200 as _pkg
from paper_2311_02909_b200 import *  # noqa: F401,F403
from paper_2311_02909_b200 import dist, errors, graph_io, pipeline, sampler, sparse  # noqa: F401

for _name in ("dist", "errors", "graph_io", "pipeline", "sampler", "sparse"):
    sys.modules[__name__ + "." + _name] = getattr(_pkg, _name)
