"""Script adapters (see scenarios.run_script) for the oracle and the product."""

import numpy as np

import oracle as O


class OracleAdapter:
    def make_store(self, cfg):
        return O.OracleStore(cfg["voxel_size"], cfg["mu"], cfg["stream_radius"])

    def stream(self, store, c):
        return store.stream(c)

    def integrate(self, store, f, p):
        new, touched, updated = store.integrate(f, p)
        keys = [int(O.pack_coords(*c)) for c in new]
        return keys, touched, updated

    def deintegrate(self, store, f, p):
        store.deintegrate(f, p)

    def gc(self, store):
        return store.garbage_collect()

    def total_weight(self, store):
        return store.total_weight()

    def correct(self, store, entries, nxt):
        n = store.correct_entries(entries)
        if nxt is not None:
            store.stream(nxt)
        return n

    def export(self, store):
        return store.export()

    def counters(self, store):
        return (store.blocks_streamed_in, store.blocks_streamed_out,
                store.sphere_relocations)


class ProductAdapter:
    """Drives paper_1709_03763_b200.volume (the CUDA path)."""

    def __init__(self, block_capacity=1 << 14):
        self.block_capacity = block_capacity

    def make_store(self, cfg):
        from paper_1709_03763_b200 import volume as V

        self.V = V
        self.cfg = V.VolumeConfig(**cfg)
        return V.TwoTierStore(block_capacity=self.block_capacity)

    def stream(self, store, c):
        return self.V.stream(store, c, self.cfg)

    def integrate(self, store, f, p):
        rec = self.V.integrate(store, f, p, self.cfg)
        keys = [int(k) for k in self.V.pack_keys(sorted(rec.new_blocks))] if rec.new_blocks else []
        return keys, rec.blocks_touched, rec.voxels_updated

    def deintegrate(self, store, f, p):
        self.V.deintegrate(store, f, p, self.cfg)

    def gc(self, store):
        return self.V.garbage_collect(store)

    def total_weight(self, store):
        return self.V.total_weight(store)

    def correct(self, store, entries, nxt):
        return self.V.correct_entries(store, entries, self.cfg, nxt)

    def export(self, store):
        return store.export()

    def counters(self, store):
        c = store.counters()
        return (c.blocks_streamed_in, c.blocks_streamed_out, c.sphere_relocations)


def logs_match(got, want, rel_weight=1e-12):
    """Compare two run_script logs: everything exact except total_weight,
    whose summation order differs (reference: Python sum over dict order)."""
    if len(got) != len(want):
        return False, "log length"
    for i, (g, w) in enumerate(zip(got, want)):
        if g["op"] != w["op"]:
            return False, f"op {i} kind"
        if g.get("error") != w.get("error"):
            return False, f"op {i} ({g['op']}) error {g.get('error')} != {w.get('error')}"
        if g["op"] == "total_weight":
            a, b = g["result"], w["result"]
            if abs(a - b) > rel_weight * max(abs(b), 1.0):
                return False, f"op {i} total_weight {a} != {b}"
        elif g.get("result") != w.get("result"):
            return False, f"op {i} ({g['op']}) result {g.get('result')} != {w.get('result')}"
        for k in ("n_blocks", "digest", "counters"):
            if g[k] != w[k]:
                return False, f"op {i} ({g['op']}) {k}: {g[k]} != {w[k]}"
    return True, ""
