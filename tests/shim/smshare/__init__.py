"""Import shim: exposes paper_2504_19516_b200 under the reference package name
`smshare`, so the reference's own test-suite (pkg/tests) runs unchanged against
this implementation.  Test infrastructure only."""

import sys

import paper_2504_19516_b200 as _impl
from paper_2504_19516_b200 import cli, engine, errors, perf_model, scheduler, workload

for _name, _mod in (("cli", cli), ("engine", engine), ("errors", errors),
                    ("perf_model", perf_model), ("scheduler", scheduler),
                    ("workload", workload)):
    sys.modules[f"{__name__}.{_name}"] = _mod

from paper_2504_19516_b200 import *  # noqa: E402,F401,F403

__version__ = _impl.__version__
