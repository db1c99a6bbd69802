"""Crafted identity collisions for the collision-check tests (tests only).

The identity chain of reading A26 is S_d = sum_{e<=d} f(c_e ^ (e+1)K ^ salt),
H_d = f(S_d) with f = fmix64, a bijection of u64 (xorshift-33 steps and odd
multipliers).  Two depth-2 paths [a1, a2] and [b1, b2] share H_2 iff their sums
S_2 agree, so for any a1, a2, b1 with a1 != b1 the key
    b2 = f^-1(f(a1^K^s) + f(a2^2K^s) - f(b1^K^s)) ^ 2K ^ s
makes a genuine 64-bit collision of two different prefixes.  f and f^-1 are
written out here from the MurmurHash3 finalizer's definition.
"""
M = (1 << 64) - 1
K = 0x9E3779B97F4A7C15
C1, C2 = 0xff51afd7ed558ccd, 0xc4ceb9fe1a85ec53


def fmix64(x):
    x ^= x >> 33
    x = (x * C1) & M
    x ^= x >> 33
    x = (x * C2) & M
    x ^= x >> 33
    return x


def fmix64_inv(y):
    y ^= y >> 33                       # xorshift by >= 32 is an involution
    y = (y * pow(C2, -1, 1 << 64)) & M
    y ^= y >> 33
    y = (y * pow(C1, -1, 1 << 64)) & M
    y ^= y >> 33
    return y


def colliding_pair(a1, a2, b1, salt=0):
    """Second key b2 such that [a1, a2] and [b1, b2] share the depth-2 identity."""
    s2 = (fmix64(a1 ^ K ^ salt) + fmix64(a2 ^ ((2 * K) & M) ^ salt) - fmix64(b1 ^ K ^ salt)) & M
    return fmix64_inv(s2) ^ ((2 * K) & M) ^ salt
