/* CRC32C (Castagnoli) oracle: the reference's slicing-by-8 table algorithm
 * (moefold/checkpoint.py:40-78, reflected polynomial 0x82F63B78, init and
 * xorout 0xFFFFFFFF, check value crc32c("123456789") = 0xE3069283) restated
 * in C so the tests can checksum megabytes quickly.
 * TEST INFRASTRUCTURE ONLY (the checker for the GPU kernel in crc32c.cu). */
#include <stddef.h>
#include <stdint.h>

static uint32_t T[8][256];
static int ready = 0;

static void make_tables(void) {
    for (int i = 0; i < 256; ++i) {        /* checkpoint.py:45-51 */
        uint32_t c = (uint32_t)i;
        for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ 0x82F63B78u : c >> 1;
        T[0][i] = c;
    }
    for (int t = 1; t < 8; ++t)            /* checkpoint.py:52-55 */
        for (int i = 0; i < 256; ++i) T[t][i] = T[0][T[t - 1][i] & 0xFF] ^ (T[t - 1][i] >> 8);
    ready = 1;
}

uint32_t oracle_crc32c(const uint8_t* d, size_t n, uint32_t crc) {
    if (!ready) make_tables();
    uint32_t c = crc ^ 0xFFFFFFFFu;        /* checkpoint.py:62-78 */
    size_t i = 0, end8 = n - (n % 8);
    for (; i < end8; i += 8) {
        c = T[7][(d[i] ^ c) & 0xFF] ^ T[6][(d[i + 1] ^ (c >> 8)) & 0xFF] ^ T[5][(d[i + 2] ^ (c >> 16)) & 0xFF] ^
            T[4][(d[i + 3] ^ (c >> 24)) & 0xFF] ^ T[3][d[i + 4]] ^ T[2][d[i + 5]] ^ T[1][d[i + 6]] ^ T[0][d[i + 7]];
    }
    for (; i < n; ++i) c = T[0][(c ^ d[i]) & 0xFF] ^ (c >> 8);
    return c ^ 0xFFFFFFFFu;
}
