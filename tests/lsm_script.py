"""Runner for the golden scripts under tests/golden/*.lsm.

Script language (one command per line, '#' lines are citations/comments):
  b <b>                      batch size
  batch <op> <op> ...        one update batch; op = I:<key>:<val> | D:<key>
  expect ... end             SPEC.md:305-307 text dump must match exactly
  packed <i> = k:v ...       level i's raw 32-bit key variables and values
  levels <i> <j> ...         the occupied levels (set bits of r)
  merged <m>                 records written by merges in the last batch,
                             in units of b (structural model only)
  lookup <k> = <v>|none
  count <k1> <k2> = <c>
  range <k1> <k2> = k:v ...  (possibly empty after '=')
  cleanup

An adapter provides: update(keys, vals, is_delete), lookup(q) -> (vals, found),
count(k1, k2), range(k1, k2) -> (offsets, keys, vals), cleanup(), r,
level(i) -> (packed keys, vals), num_levels(), and optionally merged_records.
"""
from __future__ import annotations

import glob
import os

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(__file__), "golden")


def golden_files():
    return sorted(glob.glob(os.path.join(GOLDEN_DIR, "*.lsm")))


def dump_text(ad, b) -> str:
    lines = [f"lsm b={b} r={ad.r}"]
    for i in range(ad.num_levels()):
        k, v = ad.level(i)
        if len(k) == 0:
            continue
        items = " ".join(f"{int(x) >> 1}:{'R' if int(x) & 1 else 'T'}:{int(y)}"
                         for x, y in zip(k, v))
        lines.append(f"level {i}: {items}")
    return "\n".join(lines)


def parse(path):
    cmds = []
    with open(path) as f:
        lines = [ln.rstrip("\n") for ln in f]
    i = 0
    while i < len(lines):
        ln = lines[i].strip()
        i += 1
        if not ln or ln.startswith("#"):
            continue
        if ln == "expect":
            block = []
            while lines[i].strip() != "end":
                block.append(lines[i].strip())
                i += 1
            i += 1
            cmds.append(("expect", "\n".join(block)))
        else:
            cmds.append(tuple(ln.split(" ", 1)) if " " in ln else (ln, ""))
    return cmds


def script_b(path) -> int:
    for c, a in parse(path):
        if c == "b":
            return int(a)
    raise ValueError("no b")


def run(path, make_adapter, check_structure=True):
    """Execute one script; make_adapter(b) -> adapter. Asserts on mismatch."""
    ad = None
    b = None
    merged_before = 0
    for cmd, arg in parse(path):
        where = f"{os.path.basename(path)}: {cmd} {arg}"
        if cmd == "b":
            b = int(arg)
            ad = make_adapter(b)
        elif cmd == "batch":
            keys, vals, dels = [], [], []
            for tok in arg.split():
                p = tok.split(":")
                keys.append(int(p[1]))
                vals.append(int(p[2]) if p[0] == "I" else 0)
                dels.append(1 if p[0] == "D" else 0)
            merged_before = getattr(ad, "merged_records", 0)
            ad.update(np.array(keys, np.uint32), np.array(vals, np.uint32),
                      np.array(dels, np.uint8))
        elif cmd == "expect":
            if check_structure:
                got = dump_text(ad, b)
                assert got == arg, f"{where}\n--- got\n{got}\n--- expected\n{arg}"
        elif cmd == "packed":
            if check_structure:
                lvl, rhs = arg.split("=")
                k, v = ad.level(int(lvl))
                exp = [tuple(int(x) for x in t.split(":")) for t in rhs.split()]
                got = list(zip([int(x) for x in k], [int(x) for x in v]))
                assert got == exp, f"{where}: {got} != {exp}"
        elif cmd == "levels":
            if check_structure:
                exp = [int(x) for x in arg.split()]
                got = [i for i in range(ad.num_levels()) if len(ad.level(i)[0]) > 0]
                assert got == exp, f"{where}: {got}"
                assert [i for i in range(64) if (ad.r >> i) & 1] == exp, where
        elif cmd == "merged":
            if hasattr(ad, "merged_records"):
                got = (ad.merged_records - merged_before) // b
                assert got == int(arg), f"{where}: {got}"
        elif cmd == "lookup":
            k, rhs = arg.split("=")
            v, f = ad.lookup(np.array([int(k)], np.uint32))
            rhs = rhs.strip()
            if rhs == "none":
                assert int(f[0]) == 0, f"{where}: found {int(v[0])}"
            else:
                assert int(f[0]) == 1 and int(v[0]) == int(rhs), f"{where}: {v}, {f}"
        elif cmd == "count":
            lhs, rhs = arg.split("=")
            k1, k2 = (int(x) for x in lhs.split())
            c = ad.count(np.array([k1], np.uint32), np.array([k2], np.uint32))
            assert int(c[0]) == int(rhs), f"{where}: {int(c[0])}"
        elif cmd == "range":
            lhs, rhs = arg.split("=")
            k1, k2 = (int(x) for x in lhs.split())
            off, ks, vs = ad.range(np.array([k1], np.uint32), np.array([k2], np.uint32))
            exp = [tuple(int(x) for x in t.split(":")) for t in rhs.split()]
            got = list(zip([int(x) for x in ks], [int(x) for x in vs]))
            assert got == exp, f"{where}: {got}"
            assert int(off[0]) == 0 and int(off[1]) == len(exp), where
        elif cmd == "cleanup":
            ad.cleanup()
        else:
            raise ValueError(f"unknown command {cmd}")
