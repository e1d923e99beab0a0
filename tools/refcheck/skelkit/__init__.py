"""Developer check only: `skelkit` as an alias of paper_1110_3105_b200, so the
reference's own test modules can be pointed at this package unmodified."""
import importlib
import sys

import paper_1110_3105_b200 as _pkg

for _name in ("errors", "geom", "kernels", "lowrank", "skel", "solver", "bie"):
    _m = importlib.import_module(f"paper_1110_3105_b200.{_name}")
    sys.modules[f"skelkit.{_name}"] = _m
    globals()[_name] = _m
for _k in dir(_pkg):
    if not _k.startswith("_"):
        globals().setdefault(_k, getattr(_pkg, _k))
__version__ = getattr(_pkg, "__version__", "0")
