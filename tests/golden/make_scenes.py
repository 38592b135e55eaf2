"""Writes tests/golden/scenes.json: the reference's shipped scene files
(/root/reference/proj/scenes/*.txt) parsed with the product's
pstereo_load_scene_spec, so the GPU box (which has no /root/reference) can
render the same scenes. Run here:

    python tests/golden/make_scenes.py
"""
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
import paper_2205_03133_b200 as P  # noqa: E402

SCENES = Path("/root/reference/proj/scenes")

out = {}
for f in sorted(SCENES.glob("*.txt")):
    out[f.stem] = P.load_scene_spec(f).as_dict()
(HERE / "scenes.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
print(f"wrote {len(out)} scenes")
