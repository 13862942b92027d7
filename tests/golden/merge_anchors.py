"""Merge partial anchor files written by ``make_large_anchors.py --out=...``
into tests/golden/large_anchors.json:  python tests/golden/merge_anchors.py A.json B.json"""
import json
import sys
from pathlib import Path

OUT = Path(__file__).resolve().parent / "large_anchors.json"
res = json.loads(OUT.read_text()) if OUT.exists() else {}
for f in sys.argv[1:]:
    res.update(json.loads(Path(f).read_text()))
OUT.write_text(json.dumps(res, indent=1))
print(sorted(res))
