"""The merge kernel's byte-parallel deposit (kernels.cu expand_masks /
expand_apply), restated op for op in Python, equals a bit-serial pdep: the
coin bits a disagreeing coordinate receives depend on it."""
import random

M32 = 0xFFFFFFFF


def pdep(x, m):
    r, k = 0, 0
    for i in range(32):
        if m >> i & 1:
            r |= ((x >> k) & 1) << i
            k += 1
    return r


def expand_masks(m):
    pc = (m - ((m >> 1) & 0x55555555)) & M32
    pc = ((pc & 0x33333333) + ((pc >> 2) & 0x33333333)) & M32
    pc = (pc + (pc >> 4)) & 0x0F0F0F0F
    ex = (pc * 0x01010100) & M32
    mk = ((~m) << 1) & 0xFEFEFEFE
    mv = []
    for i in range(3):
        mp = mk ^ ((mk << 1) & 0xFEFEFEFE)
        mp ^= (mp << 2) & 0xFCFCFCFC
        mp ^= (mp << 4) & 0xF0F0F0F0
        v = mp & m
        m = ((m ^ v) | (v >> (1 << i))) & M32
        mk &= ~mp & M32
        mv.append(v)
    return mv + [ex]


def byte_perm(a, b, sel):
    src = [(a >> (8 * i)) & 0xFF for i in range(4)] + [(b >> (8 * i)) & 0xFF for i in range(4)]
    return sum(src[(sel >> (4 * i)) & 7] << (8 * i) for i in range(4))


def expand_apply(x, mv):
    ex = mv[3]
    t = byte_perm(x, x >> ((ex >> 8) & 0xFF), 0x0040)
    t = byte_perm(t, x >> ((ex >> 16) & 0xFF), 0x0410)
    t = byte_perm(t, x >> (ex >> 24), 0x4210)
    for i, s in ((2, 4), (1, 2), (0, 1)):
        t = ((t & ~mv[i]) | ((t << s) & mv[i])) & M32
    return t


def test_deposit_matches_serial_pdep():
    rnd = random.Random(7)
    cases = [(rnd.getrandbits(32), rnd.getrandbits(32)) for _ in range(20000)]
    cases += [(b << (8 * p) | (rnd.getrandbits(32) & ~(0xFF << (8 * p)) & M32), rnd.getrandbits(32))
              for b in range(256) for p in range(4)]
    cases += [(0, M32), (M32, 0x12345678), (0x80000001, 3), (0x0F0F0F0F, M32)]
    for m, x in cases:
        assert expand_apply(x, expand_masks(m)) & m == pdep(x, m), (hex(m), hex(x))
