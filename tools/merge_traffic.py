"""Merge a summarize_profiles.py traffic fragment into profiles/traffic.json:
python tools/merge_traffic.py profiles/r02/traffic_fragment.json"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path = os.path.join(ROOT, "profiles", "traffic.json")
doc = json.load(open(path)) if os.path.exists(path) else {}
doc.update(json.load(open(sys.argv[1])))
with open(path, "w") as f:
    json.dump(doc, f, indent=1)
print("merged", sys.argv[1], "->", path)
