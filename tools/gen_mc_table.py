"""Emit the packed marching-cubes triangle table used by csrc/rf_mesh.cuh.

The canonical 256-case table (Lorensen & Cline's cases in Bourke's
polygoniser layout) is what the reference ships as
refusion/mc_tables.py:44-302; output parity needs the same triangle order,
so the table is read from the reference package in this container and
packed one 64-bit word per case: bits [4i, 4i+4) hold the i-th edge of the
case's triangle list (i < 15), bits 60..63 the triangle count.  The edge
masks (mc_tables.py:25-42) are not stored: a cut edge is one whose two
corners differ in sign, derived in the kernel.  tests/test_mesh.py checks
the packed words against the reference table when it is present."""

import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def reference_tables():
    for p in (os.path.join(REPO, "oracle", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "refusion")):
            sys.path.insert(0, p)
            import importlib

            return importlib.import_module("refusion.mc_tables")
    return None


def pack(case_triangles):
    words = []
    for row in case_triangles:
        edges = [int(e) for e in row if e >= 0]
        assert len(edges) % 3 == 0 and len(edges) <= 15
        w = (len(edges) // 3) << 60
        for i, e in enumerate(edges):
            w |= e << (4 * i)
        words.append(w)
    return words


def main():
    mt = reference_tables()
    if mt is None:
        sys.exit("reference package not found")
    words = pack(mt.CASE_TRIANGLES)
    print("__constant__ unsigned long long kMcTriangles[256] = {")
    for i in range(0, 256, 4):
        print("    " + ", ".join(f"0x{w:016x}ull" for w in words[i:i + 4]) + ",")
    print("};")


if __name__ == "__main__":
    main()
