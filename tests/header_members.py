"""Data-member lists of the structs in a C++ header tree (namespace mswave):
the layout contract between include/mswave/*.hpp and the reference's
proj/include/mswave/*.hpp (same members, same types, same order), used by
tests/test_header_layout.py and tools/gen_struct_golden.py."""
from __future__ import annotations

import os
import re


def _strip_comments(src: str) -> str:
    src = re.sub(r"/\*.*?\*/", " ", src, flags=re.S)
    return re.sub(r"//[^\n]*", " ", src)


def _body(src: str, open_idx: int) -> tuple[str, int]:
    depth = 0
    for i in range(open_idx, len(src)):
        if src[i] == "{":
            depth += 1
        elif src[i] == "}":
            depth -= 1
            if depth == 0:
                return src[open_idx + 1:i], i
    raise ValueError("unbalanced braces")


def _members(body: str, prefix: str, out: dict):
    # nested structs first (recorded as Outer::Inner), then removed
    while True:
        m = re.search(r"\bstruct\s+(\w+)\s*\{", body)
        if not m:
            break
        inner, end = _body(body, m.end() - 1)
        _members(inner, f"{prefix}::{m.group(1)}", out)
        stop = body.find(";", end)
        body = body[:m.start()] + body[stop + 1:]
    # drop member-function bodies and brace initialisers
    while True:
        m = re.search(r"\{", body)
        if not m:
            break
        _, end = _body(body, m.start())
        body = body[:m.start()] + ";" + body[end + 1:]
    fields = []
    for decl in body.split(";"):
        d = " ".join(decl.split())
        d = re.sub(r"^(public|private|protected)\s*:\s*", "", d)
        if not d or "(" in d or d.startswith(("using ", "enum ", "static ", "friend ", "typedef ")):
            continue
        # split "T a = x, b = y" at top-level commas
        parts, depth, cur = [], 0, ""
        for ch in d:
            if ch == "<":
                depth += 1
            elif ch == ">":
                depth -= 1
            if ch == "," and depth == 0:
                parts.append(cur)
                cur = ""
            else:
                cur += ch
        parts.append(cur)
        first = parts[0].split("=")[0].strip()
        mt = re.match(r"^(.*?)([A-Za-z_]\w*)\s*$", first)
        if not mt:
            continue
        typ = re.sub(r"\s*([<>,*&])\s*", r"\1", mt.group(1).strip())
        names = [mt.group(2)] + [p.split("=")[0].strip() for p in parts[1:]]
        for nm in names:
            fields.append([typ, nm])
    out[prefix] = fields


def struct_members(include_dir: str) -> dict:
    """{struct name: [[type, member], ...]} over every header of the tree."""
    out = {}
    for fn in sorted(os.listdir(include_dir)):
        if not fn.endswith(".hpp"):
            continue
        src = _strip_comments(open(os.path.join(include_dir, fn)).read())
        pos = 0
        while True:
            m = re.search(r"\bstruct\s+(\w+)\s*\{", src[pos:])
            if not m:
                break
            body, end = _body(src, pos + m.end() - 1)
            _members(body, m.group(1), out)
            pos = end + 1
    return out
