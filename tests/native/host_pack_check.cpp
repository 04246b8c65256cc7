// Host packer check (csrc/host_pack.cpp): pack2_rows against the 2-bit
// layout definition for V = 1..300, row strides > V, K = 2..4, and the
// gene >= K flag. Built and run by tests/test_host_pack_native.py.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include "host_pack.hpp"
int main() {
    std::mt19937 g(7); int fails = 0;
    for (int V = 1; V <= 300; V += (V < 80 ? 1 : 37)) for (int extra : {0, 3, 64}) for (int K : {2, 3, 4}) {
        const int64_t ld = V + extra, rows = 1000 + g() % 50, pld = ((V + 3) / 4 + 3) / 4 * 4;
        std::vector<uint8_t> src(rows * ld), dst(rows * pld, 0xAB);
        for (auto &x : src) x = g() % K;
        bool badset = (g() % 3 == 0); int64_t br = g() % rows; int bc = g() % V;
        if (badset) src[br * ld + bc] = K + g() % 3;
        bool ok = hs::pack2_rows(src.data(), ld, V, K, rows, dst.data(), pld);
        if (ok == badset) { printf("bad flag V=%d K=%d\n", V, K); ++fails; }
        if (badset) continue;
        for (int64_t r = 0; r < rows; ++r) for (int64_t o = 0; o < pld; ++o) {
            uint8_t e = 0; for (int q = 0; q < 4; ++q) { int64_t i = o * 4 + q; if (i < V) e |= (src[r * ld + i] & 3) << (2 * q); }
            if (dst[r * pld + o] != e) { if (fails++ < 5) printf("mismatch V=%d ld=%ld r=%ld o=%ld\n", V, (long)ld, (long)r, (long)o); }
        }
    }
    printf("fails %d\n", fails);
    return fails != 0;
}
