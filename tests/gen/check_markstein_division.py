"""Markstein division with a correctly rounded reciprocal (kcg_div in the
GPU row formation): q = RN(c r), e = RN(c - q t) (exact by FMA),
RN(q + e r) equals RN(c / t) -- checked here against exact rational
division on random and all-ones-mantissa operands (test infrastructure)."""
from fractions import Fraction as Fr
import random, struct
def fma(x,y,z): return float(Fr(x)*Fr(y)+Fr(z))
def rcp(b): return float(Fr(1)/Fr(b))
def div_m(a,b):
    r = rcp(b); q = a*r; e = fma(-q, b, a); return fma(e, r, q)
def rnd_double(rng):
    m = rng.getrandbits(52); e = rng.randint(1023-60, 1023+60)
    return struct.unpack('<d', struct.pack('<Q', (e<<52)|m))[0]
rng = random.Random(1); bad=0; N=300000
for i in range(N):
    a = rnd_double(rng); b = rnd_double(rng)
    if i % 3 == 0: b = struct.unpack('<d', struct.pack('<Q', ((1023+rng.randint(-5,5))<<52)|((1<<52)-1-rng.randint(0,3))))[0]  # near all-ones mantissa
    if i % 5 == 0: a = float(rng.randint(1, 1<<53))
    if div_m(a,b) != a/b: bad += 1
print("bad", bad, "of", N)
