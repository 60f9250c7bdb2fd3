"""Direction sharding across ranks: contiguous slices of the
leaf order in multiples of 4 patches, the rule the C runtime applies in
stamg_create (context.cu). Host-side helper shared by bench.py and tests."""


def patch_range(P: int, rank: int, world: int) -> tuple[int, int]:
    quads = (P + 3) // 4
    q0 = min(P, 4 * ((quads * rank) // world))
    q1 = min(P, 4 * ((quads * (rank + 1)) // world))
    return q0, q1
