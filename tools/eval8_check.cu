// Randomised check of the SWAR child evaluation (csrc/csv_eval8.cuh) against a
// per-child restatement of codec.py:400-457.  Host-only; build + run:
//   nvcc -O2 -std=c++17 -o /tmp/eval8_check tools/eval8_check.cu && /tmp/eval8_check
#include <cstdio>
#include <cstdlib>
#include <random>
#include "../paper_2308_16619_b200/csrc/csv_eval8.cuh"

int main(int argc, char** argv) {
    std::mt19937_64 rng(argc > 1 ? atoll(argv[1]) : 1);
    const long iters = argc > 2 ? atol(argv[2]) : 20000000;
    long fails = 0, errs = 0;
    for (long it = 0; it < iters; ++it) {
        uint64_t w = rng();
        if (it & 1) {   // bias towards ops 0..6 with small payloads
            uint64_t m = 0;
            for (int c = 0; c < 8; ++c) {
                uint32_t op = rng() % 7, st = (rng() % 8) == 0, d = rng() % 16;
                m |= (uint64_t)(op | st << 3 | d << 4) << (8 * c);
            }
            w = m;
        }
        const uint32_t pv = rng() & 0xFF, pxp = rng() & 0xFF, pyp = rng() & 0xFF, pzp = rng() & 0xFF;
        const uint32_t bf = (rng() % 4 == 0) ? (uint32_t)(rng() & 63) : 0u;
        const uint32_t plen = 1 + rng() % 256;
        const int32_t ipq = (rng() % 3 == 0) ? (int32_t)(rng() % 24) : (int32_t)(rng() % plen);
        const uint32_t nv = (rng() % 4 == 0) ? (uint32_t)(rng() % 9) : 8u;
        const uint64_t vmask = nv == 8 ? ~0ull : ((1ull << (8 * nv)) - 1ull);
        const bool leaf = rng() & 1;
        e8::Out g, gm;
        e8::eval8(w, pv, pxp, pyp, pzp, bf, ipq, plen, vmask, leaf, g);
        e8::eval8<true>(w, pv, pxp, pyp, pzp, bf, ipq, plen, vmask, leaf, gm);
        // per-child restatement
        bool err = false;
        uint32_t val[8], pend = 0, n5 = 0;
        int32_t ip = ipq;
        for (int c = 0; c < 8; ++c) {
            const uint32_t e = (uint32_t)(w >> (8 * c)) & 0xFF, op = e & 7, stop = (e >> 3) & 1, d = e >> 4;
            const bool valid = (uint32_t)c < nv;
            val[c] = 0xFFFF;
            if (op == 7) { if (valid) err = true; continue; }
            if (leaf && stop && valid) err = true;
            if (op == 0) val[c] = pv;
            else if (op <= 3) {
                const int a = op - 1;
                const bool odd = (c >> a) & 1;
                const bool bnd = (bf >> (2 * a + (odd ? 1 : 0))) & 1;
                if (bnd) { if (valid) err = true; continue; }
                if (odd) val[c] = a == 0 ? pxp : (a == 1 ? pyp : pzp);
                else pend |= op << (2 * c);
            } else if (op == 4) val[c] = (uint32_t)ip;
            else if (op == 5) {
                if (valid) ++n5;
                const int32_t idx = ip - (int32_t)d - 1;
                if (idx < 0) { if (valid) err = true; continue; }
                val[c] = (uint32_t)idx;
            } else {
                ++ip;
                if (ip >= (int32_t)plen) { if (valid) err = true; continue; }
                val[c] = (uint32_t)ip;
            }
        }
        bool bad = ((g.err != 0) != err) || g.n5 != n5;
        if (!err) {
            for (int c = 0; c < 8; ++c) {
                const uint32_t got = (uint32_t)(((uint64_t)g.vhi << 32 | g.vlo) >> (8 * c)) & 0xFF;
                if ((uint32_t)c < nv && val[c] != 0xFFFF && got != val[c]) bad = true;
            }
            if (g.pend != pend) bad = true;
            for (int c = 0; c < 8; ++c) {   // marker mode: pending children hold 252 + axis
                const uint32_t got = (uint32_t)(((uint64_t)gm.vhi << 32 | gm.vlo) >> (8 * c)) & 0xFF;
                const uint32_t a = (pend >> (2 * c)) & 3;
                if ((uint32_t)c < nv && (a ? got != 252 + a : (val[c] != 0xFFFF && got != val[c]))) bad = true;
            }
            if (gm.pend != g.pend || gm.err != g.err || gm.n5 != g.n5) bad = true;
        }
        errs += err;
        if (bad && fails++ < 10)
            printf("MISMATCH w=%016llx pv=%u px=%u py=%u pz=%u bf=%u ipq=%d plen=%u nv=%u leaf=%d: err %u/%d pend %x/%x n5 %u/%u\n",
                   (unsigned long long)w, pv, pxp, pyp, pzp, bf, ipq, plen, nv, (int)leaf, g.err, (int)err, g.pend, pend,
                   g.n5, n5);
    }
    printf("%ld cases, %ld with errors, %ld mismatches\n", iters, errs, fails);
    return fails != 0;
}
