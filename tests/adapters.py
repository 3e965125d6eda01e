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
