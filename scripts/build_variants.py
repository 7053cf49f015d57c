"""Build libtomo A/B variants (compile-time -D knobs) next to the default library:
    python scripts/build_variants.py name:DEF1,DEF2 name2:DEF3 ...
-> paper_2104_12282_b200/lib/<name>.so (timing: TOMO_LIB_PATH=... python scripts/time_apply.py)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_12282_b200 import build  # noqa: E402

for spec in sys.argv[1:]:
    name, _, defs = spec.partition(":")
    out = os.path.join(os.path.dirname(build.LIB), name + ".so")
    build.build(force=True, defines=[d for d in defs.split(",") if d], out=out)
    print(out)
