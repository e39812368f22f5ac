"""A/B timing of two libpidb builds on the same box:
python tools/ab_k5.py LIB N RES reps  (LIB: path of the .so to load)"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2512_15187_b200 import _native as N  # noqa: E402

N.load(sys.argv[1])
sys.argv = [sys.argv[0]] + sys.argv[2:]
exec(open(Path(__file__).with_name("prof_k5.py")).read())
