// Counter-keyed uniforms on device: numpy SeedSequence -> PCG64 -> double.
//
// Bit-exact restatement of the generator the reference builds per key,
// default_rng(SeedSequence(entropy=(seed, seq_id, role, counter)))
// (ref:sampling.py:53-66); the integer spec is oracle/rng.py.  Draw n of a
// key is (next64 >> 11) * 2^-53 (ref:sampling.py:107-115 consumes it).
#pragma once
#include "common.cuh"

namespace bass {

struct Pcg64 {
    unsigned __int128 state, inc;
};

BASS_DEV uint32_t ss_hashmix(uint32_t value, uint32_t& hc) {
    value ^= hc;
    hc *= 0x931E8875u;
    value *= hc;
    return value ^ (value >> 16);
}
BASS_DEV uint32_t ss_mix(uint32_t x, uint32_t y) {
    uint32_t r = 0xCA01F9DDu * x - 0x4973F715u * y;
    return r ^ (r >> 16);
}

// append the little-endian uint32 words of a non-negative integer
BASS_DEV int ss_words(uint64_t x, uint32_t* w, int n) {
    if (x == 0) { w[n++] = 0; return n; }
    while (x) { w[n++] = uint32_t(x); x >>= 32; }
    return n;
}

BASS_DEV Pcg64 pcg64_from_key(uint64_t seed, uint64_t sid, uint32_t role, uint64_t ctr) {
    uint32_t ent[8];
    int n = 0;
    n = ss_words(seed, ent, n);
    n = ss_words(sid, ent, n);
    n = ss_words(role, ent, n);
    n = ss_words(ctr, ent, n);
    uint32_t pool[4];
    uint32_t hc = 0x43B0D7E5u;
#pragma unroll
    for (int i = 0; i < 4; ++i) pool[i] = ss_hashmix(i < n ? ent[i] : 0u, hc);
#pragma unroll
    for (int s = 0; s < 4; ++s)
#pragma unroll
        for (int d = 0; d < 4; ++d)
            if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], hc));
    for (int s = 4; s < n; ++s)
#pragma unroll
        for (int d = 0; d < 4; ++d) pool[d] = ss_mix(pool[d], ss_hashmix(ent[s], hc));
    uint32_t words[8];
    uint32_t hb = 0x8B51F9DDu;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        uint32_t v = pool[i & 3] ^ hb;
        hb *= 0x58F38DEDu;
        v *= hb;
        words[i] = v ^ (v >> 16);
    }
    uint64_t u64[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) u64[i] = uint64_t(words[2 * i]) | (uint64_t(words[2 * i + 1]) << 32);
    const unsigned __int128 mult =
        ((unsigned __int128)2549297995355413924ull << 64) | 4865540595714422341ull;
    unsigned __int128 initstate = ((unsigned __int128)u64[0] << 64) | u64[1];
    unsigned __int128 initseq = ((unsigned __int128)u64[2] << 64) | u64[3];
    Pcg64 g;
    g.inc = (initseq << 1) | 1;
    g.state = g.inc;              // 0 * mult + inc
    g.state += initstate;
    g.state = g.state * mult + g.inc;
    return g;
}

BASS_DEV uint64_t pcg64_next(Pcg64& g) {
    const unsigned __int128 mult =
        ((unsigned __int128)2549297995355413924ull << 64) | 4865540595714422341ull;
    g.state = g.state * mult + g.inc;
    uint64_t x = uint64_t(g.state >> 64) ^ uint64_t(g.state);
    uint32_t rot = uint32_t(g.state >> 122);
    return (x >> rot) | (x << ((64 - rot) & 63));
}

BASS_DEV double pcg64_double(Pcg64& g) {
    return double(pcg64_next(g) >> 11) * (1.0 / 9007199254740992.0);
}

// Benchmark-harness hash (aligned-draft override and device weight init):
// splitmix64 finaliser over a combined key.  Not a reference RNG.
BASS_DEV uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

}  // namespace bass
