"""CPU ORACLE backend of the distributed BH protocol -- TEST INFRASTRUCTURE ONLY.

bh_dist.DistBH runs its host protocol (sample sort, straddling cubes, branch
summaries, LET, tree assembly) unchanged and calls this backend where the
product calls libgcharm.so: octant keys (restated from bh_build.cu bb_keys),
the forced-split local build (orc_build_tree_forced: the reference's
build_bucket_tree, nbody.py:78-143, plus forced cubes) and the walk + forces
over the assembled tree (build_interaction_lists / eval_forces restated,
nbody.py:146-250).  Used only by tests/test_bh_dist_cpu.py.
"""
import numpy as np

from . import oracle as orc


class OracleBackend:
    def keys(self, pos, box):
        return orc.octant_keys(pos, box)

    def local_tree(self, pos, mass, bucket, box, forced):
        t = orc.build_bucket_tree(pos, mass, bucket, box=box, forced=forced)
        return dict(center=t.center, half=t.half, mass=t.mass, com=t.com, first_child=t.first_child,
                    n_child=t.n_child, pstart=t.pstart, pcount=t.pcount, buckets=t.buckets, pidx=t.pidx)

    def step(self, tree, own, theta, g, eps, want_lists):
        dim = tree["center"].shape[1]
        nn = len(tree["half"])
        pstart = np.zeros(nn, np.int64)
        pstart[:] = tree["pstart"]
        ot = orc.OracleTree(dim=dim, center=tree["center"], half=tree["half"], mass=tree["mass"], com=tree["com"],
                            first_child=tree["first_child"], n_child=tree["n_child"].astype(np.int32),
                            pstart=pstart, pcount=tree["pcount"], buckets=tree["buckets"], pidx=tree["order"])
        ol = orc.build_interaction_lists(ot, theta, bucket_range=own)
        f = orc.eval_forces(ot, ol, tree["pos"], tree["pmass"], g, eps, bucket_range=own)
        return f, ((ol.ptr, ol.ids, ol.kind, ol.item_count) if want_lists else None)
