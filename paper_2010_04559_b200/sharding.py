"""Direction sharding across ranks.

Contexts without a hierarchy (config 5) give each rank whole orbits of the
angular mesh's reflection symmetry group (`stamg.shard_patches`, the rule
stamg_create applies), so every rank can fold its own scatter; `patch_range` is
the fallback for meshes without symmetry: contiguous slices of the leaf order in
multiples of 4 patches. `runs` splits a patch set into contiguous ranges."""


def patch_range(P: int, rank: int, world: int) -> tuple[int, int]:
    quads = (P + 3) // 4
    q0 = min(P, 4 * ((quads * rank) // world))
    q1 = min(P, 4 * ((quads * (rank + 1)) // world))
    return q0, q1


def runs(patches) -> list[tuple[int, int]]:
    """Maximal contiguous ranges [q0, q1) of an ascending patch list."""
    out = []
    for q in patches:
        q = int(q)
        if out and out[-1][1] == q:
            out[-1] = (out[-1][0], q + 1)
        else:
            out.append((q, q + 1))
    return out
