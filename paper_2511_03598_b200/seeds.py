"""Seed derivation of the reference (proj/core/src/rng.cpp:11-17,75-78):
derive_seed(seed, tag) = splitmix64(seed ^ (0xd1342543de82ef95 * (tag + 1)))."""

_M = (1 << 64) - 1


def splitmix64(x: int):
    x = (x + 0x9E3779B97F4A7C15) & _M
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M
    return z ^ (z >> 31), x


def derive_seed(seed: int, tag: int) -> int:
    s = (seed ^ ((0xD1342543DE82EF95 * (tag + 1)) & _M)) & _M
    return splitmix64(s)[0]
