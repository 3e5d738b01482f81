// Host-side bounds and injectivity checks of the tiled fill's shadow layout
// (rotor_common.cuh): every cell row and quad-minimum row of A32 / C32 lies in
// its table and no two share a row; every operand block the pruned middle
// copies (one ring stage: KC consecutive splits) lies inside the table; the
// columns the leaves write stay within [0, S].  Built and run by
// tests/test_layout.py (no GPU: only the __host__ __device__ index functions
// are called).  A bounds check of our own next to compute-sanitizer.
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#include "rotor_common.cuh"

using namespace rotor;

static int fails = 0;
#define CHECK(c, ...)                                   \
    do {                                                \
        if (!(c)) {                                     \
            if (fails++ < 20) fprintf(stderr, __VA_ARGS__); \
        }                                               \
    } while (0)

static void check(int L) {
    const int n = L + 1, nb = (n + kTB - 1) / kTB;
    const int64_t ra = shadow_rows_a(n), rc = shadow_rows_c(n);
    std::vector<unsigned char> ua(ra, 0), uc(rc, 0);
    // A32 cells: A(s, c), s <= c <= n - 1
    for (int c = 1; c < n; c++)
        for (int s = 1; s <= c; s++) {
            const int64_t r = srow_a(n, s, c);
            CHECK(r >= 0 && r < ra, "L=%d A row (%d,%d) = %lld out of [0,%lld)\n", L, s, c, (long long)r, (long long)ra);
            if (r >= 0 && r < ra) CHECK(!ua[r]++, "L=%d A row (%d,%d) reused\n", L, s, c);
        }
    // A32 quad minima: block I, group g, column c of the block's columns
    for (int I = 0; I < nb; I++)
        for (int c = kTB * I + 1; c <= n; c++)
            for (int g = 0; g < 8; g++) {
                const int64_t r = sa_col(n, I, c) + kQuad + g;
                CHECK(r >= 0 && r < ra, "L=%d QA (%d,%d,%d) out of range\n", L, I, g, c);
                if (r >= 0 && r < ra) CHECK(!ua[r]++, "L=%d QA (%d,%d,%d) collides\n", L, I, g, c);
            }
    // C32 cells: C(s, t), s <= t <= n
    for (int s = 1; s <= n; s++)
        for (int t = s; t <= n; t++) {
            const int64_t r = srow_c(s, t);
            CHECK(r >= 0 && r < rc, "L=%d C row (%d,%d) out of range\n", L, s, t);
            if (r >= 0 && r < rc) CHECK(!uc[r]++, "L=%d C row (%d,%d) reused\n", L, s, t);
        }
    // C32 quad minima: block J, row s <= min(n, 32 (J + 1)), group g
    for (int J = 0; J < nb; J++)
        for (int s = 1; s <= n && s <= kTB * (J + 1); s++)
            for (int g = 0; g < 8; g++) {
                const int64_t r = sc_row(J, s) + kQuad + g;
                CHECK(r >= 0 && r < rc, "L=%d QC (%d,%d,%d) out of range\n", L, J, s, g);
                if (r >= 0 && r < rc) CHECK(!uc[r]++, "L=%d QC (%d,%d,%d) collides\n", L, J, s, g);
            }
    // the middle's ring stages: tile (I, J), J >= I + 2, splits sp0 .. sp0 + KC - 1
    const int KC = 4;
    for (int I = 0; I < nb; I++)
        for (int J = I + 2; J < nb; J++) {
            const int i0 = kTB * I + 1, j0 = kTB * J + 1;
            CHECK((j0 - 1 - (i0 + kTB) + 1) % KC == 0, "L=%d tile (%d,%d): split range not KC-aligned\n", L, I, J);
            for (int sp0 = i0 + kTB; sp0 + KC - 1 <= j0 - 1; sp0 += KC) {
                const int64_t a0 = sa_col(n, I, sp0 - 1), c0 = sc_row(J, sp0);
                CHECK(a0 >= 0 && a0 + (int64_t)KC * kSR <= ra, "L=%d A stage (%d,%d,%d) out of range\n", L, I, J, sp0);
                CHECK(c0 >= 0 && c0 + (int64_t)KC * kSR <= rc, "L=%d C stage (%d,%d,%d) out of range\n", L, I, J, sp0);
                for (int k = 0; k < KC; k++) {  // contiguous: split k's rows start k * kSR in
                    CHECK(sa_col(n, I, sp0 + k - 1) == a0 + k * kSR, "L=%d A stage not contiguous\n", L);
                    CHECK(sc_row(J, sp0 + k) == c0 + k * kSR, "L=%d C stage not contiguous\n", L);
                    for (int r = 0; r < kTB; r++) {  // the box's cell rows are the cells it names
                        if (i0 + r <= sp0 + k - 1) CHECK(srow_a(n, i0 + r, sp0 + k - 1) == a0 + k * kSR + r, "A box row\n");
                        if (j0 + r <= n) CHECK(srow_c(sp0 + k, j0 + r) == c0 + k * kSR + r, "C box row\n");
                    }
                }
            }
        }
    // shadow_index: the m-chunked index of the last row and column stays inside rows x pitch
    for (int S : {1, 31, 32, 33, 500, 4000}) {
        const int64_t pitch = ((int64_t)kPad + S + 1 + 31) / 32 * 32;
        const int last_chunk_col = (int)((S / 32) * 32 + 31);
        CHECK(last_chunk_col < pitch, "S=%d: chunk past the pitch\n", S);
        CHECK(shadow_index(ra, ra - 1, last_chunk_col) < ra * pitch, "S=%d: A index past the table\n", S);
        CHECK(shadow_index(rc, rc - 1, last_chunk_col) < rc * pitch, "S=%d: C index past the table\n", S);
    }
}

int main(int argc, char **argv) {
    int Ls[] = {1, 2, 30, 31, 32, 33, 63, 64, 65, 95, 96, 97, 100, 130, 230, 300};
    for (int L : Ls) check(L);
    if (argc > 1) check(atoi(argv[1]));
    if (fails) {
        fprintf(stderr, "%d layout check(s) failed\n", fails);
        return 1;
    }
    printf("layout ok\n");
    return 0;
}
