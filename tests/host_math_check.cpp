// Host build of the kernel's byte-SWAR and cut-point helpers (csrc/dmsgm_math.cuh),
// checked against the literal per-pixel predicate of App. E P:657 (reading R14).
// Built and run by tests/test_host_math.py with g++ -ffp-contract=off.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <random>

#include "dmsgm_math.cuh"

using namespace dmsgm;

static long long g_slow = 0;

static int check_interval(float mu, float T, float r, long long* fails) {
    // the kernel's composition: fast form, falling back to the tested form (short form
    // without emptiness tests only when T >= 0.25)
    bool slow = false;
    Interval iv = bg_interval_fast(mu, T, r, !(T >= 0.25f), &slow);
    if (slow) {
        ++g_slow;
        iv = bg_interval(mu, T, r, !(T >= 0.25f));
    }
    const uint32_t ka = key_a(iv.a) * 0x00010001u, kb = key_b(iv.b) * 0x00010001u;
    uint8_t got[256];
    for (int I = 0; I < 256; I += 4) {
        uint32_t px = (uint32_t)I | ((uint32_t)(I + 1) << 8) | ((uint32_t)(I + 2) << 16) | ((uint32_t)(I + 3) << 24);
        uint32_t m = mask_word(lanes_lo(px), lanes_hi(px), ka, kb, ka, kb);
        for (int j = 0; j < 4; ++j) got[I + j] = (m >> (8 * j)) & 0xFF;
    }
    int bad = 0;
    for (int I = 0; I < 256; ++I) {
        const uint8_t expect = fg_pred((float)I, mu, T) ? 255 : 0;
        if (got[I] != expect) ++bad;
    }
    if (bad) {
        if (*fails < 10)
            printf("MISMATCH mu=%.9g T=%.9g r=%.9g a=%d b=%d bad=%d\n", mu, T, r, iv.a, iv.b, bad);
        ++*fails;
    }
    return bad;
}

int main(int argc, char** argv) {
    long long trials = argc > 1 ? atoll(argv[1]) : 2000000;
    long long fails = 0;
    // 1) lane primitives: every (pixel, a, b) in every byte position, mixed per-lane keys
    std::mt19937 rng(1234);
    long long swar_bad = 0;
    for (int a = 0; a <= 256; ++a)
        for (int b = 0; b < 256; b += (a == 256 ? 255 : 1))
            for (int pos = 0; pos < 4; ++pos) {
                const int I = (int)(rng() & 0xFF);
                uint32_t px = rng();
                px = (px & ~(0xFFu << (8 * pos))) | ((uint32_t)I << (8 * pos));
                // lane of byte pos gets keys (a, b); other lanes get random keys
                uint32_t ka[2], kb[2];
                for (int h = 0; h < 2; ++h) {
                    uint32_t k0 = key_a((int)(rng() % 257)), k1 = key_a((int)(rng() % 257));
                    uint32_t m0 = key_b((int)(rng() % 256)), m1 = key_b((int)(rng() % 256));
                    ka[h] = k0 | (k1 << 16);
                    kb[h] = m0 | (m1 << 16);
                }
                const int h = pos / 2, l = pos % 2;
                ka[h] = (ka[h] & ~(0xFFFFu << (16 * l))) | (key_a(a) << (16 * l));
                kb[h] = (kb[h] & ~(0xFFFFu << (16 * l))) | (key_b(b) << (16 * l));
                const uint32_t m = mask_word(lanes_lo(px), lanes_hi(px), ka[0], kb[0], ka[1], kb[1]);
                const uint32_t got = (m >> (8 * pos)) & 0xFF;
                const uint32_t expect = (a <= 255 && I >= a && I <= b) ? 0u : 0xFFu;
                if (got != expect) ++swar_bad;
            }
    printf("swar_bad %lld\n", swar_bad);

    // 2) background intervals: random and adversarial (mu, T), sqrt estimates off by a few ulp
    std::uniform_real_distribution<float> U(0.f, 1.f);
    const float thetas[] = {4.f, 1.f, 9.f, 2.5f, 16.f};
    for (long long t = 0; t < trials; ++t) {
        float mu;
        const int kind = (int)(t % 6);
        if (kind == 0) mu = 255.f * U(rng);
        else if (kind == 1) mu = (float)(int)(256.f * U(rng));                  // integer mean
        else if (kind == 2) mu = (float)(int)(255.f * U(rng)) + 0.5f;           // half-integer
        else if (kind == 3) mu = nextafterf((float)(int)(256.f * U(rng)), U(rng) < 0.5f ? 0.f : 300.f);
        else if (kind == 4) mu = U(rng) < 0.5f ? 255.f * U(rng) * U(rng) * U(rng) : 255.f - 255.f * U(rng) * U(rng) * U(rng);
        else mu = 255.00003f * U(rng);
        if (mu > 255.f && kind != 5) mu = 255.f;
        float var;
        const int vk = (int)((t / 6) % 4);
        if (vk == 0) var = expf(logf(1e-4f) + (logf(1e6f) - logf(1e-4f)) * U(rng));
        else if (vk == 1) var = 0.25f * U(rng);
        else if (vk == 2) var = (float)(int)(2000.f * U(rng)) * 0.25f;
        else var = 65025.f * U(rng);
        const float theta = thetas[(t / 24) % 5];
        float T = theta * (var > 0.25f ? var : 0.25f);
        if ((t & 7) == 7) {
            // T exactly at fl(fl(k - mu)^2) for some k, or one ulp either side
            int k = (int)(256.f * U(rng));
            float d = f_sub((float)k, mu);
            T = f_mul(d, d);
            int side = (int)(3.f * U(rng));
            if (side == 1) T = nextafterf(T, 0.f);
            if (side == 2) T = nextafterf(T, INFINITY);
            if (!(T > 0.f)) T = 1e-6f;
        }
        const float sq = sqrtf(T);
        const float r = sq * (1.0f + (U(rng) - 0.5f) * 6e-7f);   // MUFU.RSQ-class estimate
        check_interval(mu, T, r, &fails);
        if (T >= 0.25f) {   // the full form must agree too
            const Interval a1 = bg_interval(mu, T, r, true), a2 = bg_interval(mu, T, r, false);
            if (a1.a != a2.a || (a1.a <= 255 && a1.b != a2.b)) ++fails;
        }
    }
    printf("interval_fails %lld of %lld (slow path %lld)\n", fails, trials, g_slow);
    return (swar_bad || fails) ? 1 : 0;
}
