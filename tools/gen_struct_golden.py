"""Regenerate tests/golden/reference_struct_members.json from the reference's
headers (/root/reference/proj/include/mswave, read here only; the fixture
travels, the reference does not)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from tests.header_members import struct_members  # noqa: E402

REF = "/root/reference/proj/include/mswave"

if __name__ == "__main__":
    members = struct_members(REF)
    out = os.path.join(ROOT, "tests", "golden", "reference_struct_members.json")
    with open(out, "w") as f:
        json.dump({"source": "proj/include/mswave/*.hpp", "structs": members}, f, indent=1, sort_keys=True)
    print(out, len(members), "structs")
