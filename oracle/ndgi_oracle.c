/*
 * ndgi_oracle.c -- plain, slow, obviously-correct CPU oracle for the NDGI
 * tile-decode hot path (arXiv 2604.12625).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA
 * path under paper_2604_12625_b200/ and includes nothing from it.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n.  Readings R1..R20
 * are listed in DESIGN.md section "Readings of the paper".
 *
 * What it computes (Eq. 3/4):
 *   I(u,v,t) = G_Phi(V_uvt, V_uv, V_ut, V_vt, gamma(t))
 * with every feature fetched from its stored format (BC7 blocks decoded
 * from scratch on every tap), sampled bilinearly at
 * texel centres with clamp (R1), trilinearly for F_uvt (R4), an fp64 MLP
 * with GELU on the hidden layers and a linear output, weights
 * stored as f16 (R11).
 *
 * Pins (tests/test_oracle_*.py): BC7 (and BC1/BC3/BC4/BC5) against
 * Pillow's independent BCn decoder and hand vectors; samplers against torch grid_sample; MLP against
 * torch F.linear/F.gelu in fp64; gamma against closed forms;
 * border against torch F.pad(mode="reflect"); the whole pipeline against a
 * composition of those library routines.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

/* ------------------------------------------------------------------ */
/* Layout (the oracle's own struct; mirrors the meaning, not the code, of
 * include/ndgi.h).                                                     */
/* ------------------------------------------------------------------ */
enum { OR_FMT_BC7 = 0, OR_FMT_U8 = 1, OR_FMT_F16 = 2, OR_FMT_BC1 = 3, OR_FMT_BC3 = 4, OR_FMT_BC5 = 5 };
enum { OR_GELU_ERF = 0, OR_GELU_TANH = 1 };
enum { OR_BORDER_MIRROR = 0, OR_BORDER_EVAL_CLAMP = 1 };

typedef struct {
    int32_t num_tiles, atlases, tiles_x, tiles_y;
    int32_t core, border;
    int32_t uv_res, uvt_res, uvt_depth, line_res, line_t;
    int32_t hidden;
    int32_t fmt_uv, fmt_uvt, fmt_line;
    int32_t gelu, border_mode;
} oracle_layout;

typedef struct {
    const uint8_t *uv, *uvt, *ut, *vt; /* raw bytes, per-tile dense */
    const uint16_t *mlp;               /* f16 bit patterns */
} oracle_maps;

/* ------------------------------------------------------------------ */
/* f16 -> double, exact (IEEE 754 binary16).                           */
/* ------------------------------------------------------------------ */
double oracle_half_to_double(uint16_t h)
{
    int s = (h >> 15) & 1, e = (h >> 10) & 31, m = h & 1023;
    double v;
    if (e == 0)       v = ldexp((double)m, -24);               /* subnormal */
    else if (e == 31) v = m ? NAN : INFINITY;
    else              v = ldexp((double)(m + 1024), e - 25);
    return s ? -v : v;
}

/* ------------------------------------------------------------------ */
/* BC7 (BPTC) block decoder.  Definition: D3D11 functional spec, BC7
 * section / Khronos Data Format spec, BPTC.  The paper stores F_uv and
 * every t-slice of F_uvt as BC7 and describes the per-block
 * endpoint interpolation c_p = (1-w_p) e1 + w_p e2 with multi-partition
 * modes.                                                   */
/* ------------------------------------------------------------------ */

/* per-mode parameters: subsets, partition bits, rotation bits, index
 * selection bits, colour bits, alpha bits, per-endpoint p-bits, shared
 * (per-subset) p-bits, primary index bits, secondary index bits        */
typedef struct { int ns, pb, rb, isb, cb, ab, epb, spb, ib, ib2; } bc7_mode_info;
static const bc7_mode_info BC7_MODES[8] = {
    {3, 4, 0, 0, 4, 0, 1, 0, 3, 0},
    {2, 6, 0, 0, 6, 0, 0, 1, 3, 0},
    {3, 6, 0, 0, 5, 0, 0, 0, 2, 0},
    {2, 6, 0, 0, 7, 0, 1, 0, 2, 0},
    {1, 0, 2, 1, 5, 6, 0, 0, 2, 3},
    {1, 0, 2, 0, 7, 8, 0, 0, 2, 2},
    {1, 0, 0, 0, 7, 7, 1, 0, 4, 0},
    {2, 6, 0, 0, 5, 5, 1, 0, 2, 0},
};

/* Two-subset partitions, written as in the D3D11 spec: one digit per texel
 * in raster order (texel 0 first), the digit is the subset.             */
static const char *const BC7_P2[64] = {
    "0011001100110011", "0001000100010001", "0111011101110111", "0001001100110111",
    "0000000100010011", "0011011101111111", "0001001101111111", "0000000100110111",
    "0000000000010011", "0011011111111111", "0000000101111111", "0000000000010111",
    "0001011111111111", "0000000011111111", "0000111111111111", "0000000000001111",
    "0000100011101111", "0111000100000000", "0000000010001110", "0111001100010000",
    "0011000100000000", "0000100011001110", "0000000010001100", "0111001100110001",
    "0011000100010000", "0000100010001100", "0110011001100110", "0011011001101100",
    "0001011111101000", "0000111111110000", "0111000110001110", "0011100110011100",
    "0101010101010101", "0000111100001111", "0101101001011010", "0011001111001100",
    "0011110000111100", "0101010110101010", "0110100101101001", "0101101010100101",
    "0111001111001110", "0001001111001000", "0011001001001100", "0011101111011100",
    "0110100110010110", "0011110011000011", "0110011010011001", "0000011001100000",
    "0100111001000000", "0010011100100000", "0000001001110010", "0000010011100100",
    "0110110010010011", "0011011011001001", "0110001110011100", "0011100111000110",
    "0110110011001001", "0110001100111001", "0111111010000001", "0001100011100111",
    "0000111100110011", "0011001111110000", "0010001011101110", "0100010001110111",
};

/* Three-subset partitions, same notation. */
static const char *const BC7_P3[64] = {
    "0011001102212222", "0001001122112221", "0000200122112211", "0222002200110111",
    "0000000011221122", "0011001100220022", "0022002211111111", "0011001122112211",
    "0000000011112222", "0000111111112222", "0000111122222222", "0012001200120012",
    "0112011201120112", "0122012201220122", "0011011211221222", "0011200122002220",
    "0001001101121122", "0111001120012200", "0000112211221122", "0022002200221111",
    "0111011102220222", "0001000122212221", "0000001101220122", "0000110022102210",
    "0122012200110000", "0012001211222222", "0110122112210110", "0000011012211221",
    "0022110211020022", "0110011020022222", "0011012201220011", "0000200022112221",
    "0000000211221222", "0222002200120011", "0011001200220222", "0120012001200120",
    "0000111122220000", "0120120120120120", "0120201212010120", "0011220011220011",
    "0011112222000011", "0101010122222222", "0000000021212121", "0022112200221122",
    "0022001100220011", "0220122102201221", "0101222222220101", "0000212121212121",
    "0101010101012222", "0222011102220111", "0002111200021112", "0000211221122112",
    "0222011101110222", "0002111211120002", "0110011001102222", "0000000021122112",
    "0110011022222222", "0022001100110022", "0022112211220022", "0000000000002112",
    "0002000100020001", "0222122202221222", "0101222222222222", "0111201122012220",
};

/* Anchor ("fix-up") texels.  Subset 0's anchor is texel 0. */
static const int BC7_A2[64] = {
    15,15,15,15,15,15,15,15, 15,15,15,15,15,15,15,15,
    15, 2, 8, 2, 2, 8, 8,15,  2, 8, 2, 2, 8, 8, 2, 2,
    15,15, 6, 8, 2, 8,15,15,  2, 8, 2, 2, 2,15,15, 6,
     6, 2, 6, 8,15,15, 2, 2, 15,15,15,15,15, 2, 2,15,
};
static const int BC7_A3a[64] = {
     3, 3,15,15, 8, 3,15,15,  8, 8, 6, 6, 6, 5, 3, 3,
     3, 3, 8,15, 3, 3, 6,10,  5, 8, 8, 6, 8, 5,15,15,
     8,15, 3, 5, 6,10, 8,15, 15, 3,15, 5,15,15,15,15,
     3,15, 5, 5, 5, 8, 5,10,  5,10, 8,13,15,12, 3, 3,
};
static const int BC7_A3b[64] = {
    15, 8, 8, 3,15,15, 3, 8, 15,15,15,15,15,15,15, 8,
    15, 8,15, 3,15, 8,15, 8,  3,15, 6,10,15,15,10, 8,
    15, 3,15,10,10, 8, 9,10,  6,15, 8,15, 3, 6, 6, 8,
    15, 3,15,15,15,15,15,15, 15,15,15,15, 3,15,15, 8,
};

/* Interpolation weights, D3D11 spec aWeight2/3/4. */
static const int BC7_W2[4]  = {0, 21, 43, 64};
static const int BC7_W3[8]  = {0, 9, 18, 27, 37, 46, 55, 64};
static const int BC7_W4[16] = {0, 4, 9, 13, 17, 21, 26, 30, 34, 38, 43, 47, 51, 55, 60, 64};

int oracle_bc7_weight(int bits, int index)
{
    if (bits == 2) return BC7_W2[index & 3];
    if (bits == 3) return BC7_W3[index & 7];
    if (bits == 4) return BC7_W4[index & 15];
    return -1;
}

/* partition table digit for (number of subsets, partition, texel) */
int oracle_bc7_subset(int ns, int part, int texel)
{
    if (ns == 1) return 0;
    if (ns == 2) return BC7_P2[part][texel] - '0';
    return BC7_P3[part][texel] - '0';
}

int oracle_bc7_anchor(int ns, int part, int subset)
{
    if (subset == 0) return 0;
    if (ns == 2) return BC7_A2[part];
    return subset == 1 ? BC7_A3a[part] : BC7_A3b[part];
}

/* LSB-first bit reader over the 16-byte block */
typedef struct { const uint8_t *b; int pos; } bitreader;
static int take(bitreader *r, int n)
{
    int v = 0;
    for (int i = 0; i < n; ++i) {
        int bit = (r->b[r->pos >> 3] >> (r->pos & 7)) & 1;
        v |= bit << i;
        r->pos++;
    }
    return v;
}

/* expand an n-bit endpoint component to 8 bits by bit replication */
static int expand8(int v, int n)
{
    if (n >= 8) return v;
    v <<= (8 - n);
    return v | (v >> n);
}

static int interp(int e0, int e1, int w) { return ((64 - w) * e0 + w * e1 + 32) >> 6; }

/* Decodes one 128-bit block into 16 RGBA8 texels (texel = 4*row + col).
 * Returns the number of bits consumed (128 for modes 0..7, 8 for the
 * reserved mode-8 encoding, which decodes to all zeros, reading R9).   */
int oracle_bc7_decode_block(const uint8_t blk[16], uint8_t out[64])
{
    bitreader r = {blk, 0};
    int mode = 0;
    while (mode < 8 && take(&r, 1) == 0) mode++;
    if (mode == 8) { memset(out, 0, 64); return r.pos; }
    const bc7_mode_info *mi = &BC7_MODES[mode];
    int part = take(&r, mi->pb);
    int rot = take(&r, mi->rb);
    int isel = take(&r, mi->isb);

    int ep[3][2][4];        /* [subset][endpoint][channel] raw field value */
    int nbits[4];           /* bits per channel before p-bit */
    int ne = mi->ns * 2;
    for (int c = 0; c < 3; ++c) {
        nbits[c] = mi->cb;
        for (int e = 0; e < ne; ++e) ep[e / 2][e % 2][c] = take(&r, mi->cb);
    }
    if (mi->ab > 0) {
        nbits[3] = mi->ab;
        for (int e = 0; e < ne; ++e) ep[e / 2][e % 2][3] = take(&r, mi->ab);
    } else {
        nbits[3] = 0;
    }
    /* p-bits: appended as the LSB of every channel of the endpoint */
    int pbit[3][2] = {{0, 0}, {0, 0}, {0, 0}};
    int has_p = 0;
    if (mi->epb) {
        has_p = 1;
        for (int e = 0; e < ne; ++e) pbit[e / 2][e % 2] = take(&r, 1);
    } else if (mi->spb) {
        has_p = 1;
        for (int s = 0; s < mi->ns; ++s) { int p = take(&r, 1); pbit[s][0] = p; pbit[s][1] = p; }
    }
    int col[3][2][4];       /* expanded 8-bit endpoints */
    for (int s = 0; s < mi->ns; ++s)
        for (int e = 0; e < 2; ++e)
            for (int c = 0; c < 4; ++c) {
                if (c == 3 && nbits[3] == 0) { col[s][e][c] = 255; continue; }
                int v = ep[s][e][c], n = nbits[c];
                if (has_p) { v = (v << 1) | pbit[s][e]; n += 1; }
                col[s][e][c] = expand8(v, n);
            }
    /* primary indices */
    int idx1[16], idx2[16];
    for (int i = 0; i < 16; ++i) {
        int s = oracle_bc7_subset(mi->ns, part, i);
        int n = mi->ib - (i == oracle_bc7_anchor(mi->ns, part, s) ? 1 : 0);
        idx1[i] = take(&r, n);
    }
    /* secondary indices (modes 4 and 5); anchor = texel 0 */
    if (mi->ib2 > 0)
        for (int i = 0; i < 16; ++i) idx2[i] = take(&r, mi->ib2 - (i == 0 ? 1 : 0));

    for (int i = 0; i < 16; ++i) {
        int s = oracle_bc7_subset(mi->ns, part, i);
        int rgba[4];
        if (mi->ib2 == 0) {
            int w = oracle_bc7_weight(mi->ib, idx1[i]);
            for (int c = 0; c < 4; ++c) rgba[c] = interp(col[s][0][c], col[s][1][c], w);
        } else {
            /* mode 4: index-selection bit swaps which array drives colour */
            int cbits = mi->ib, abits = mi->ib2, ci = idx1[i], ai = idx2[i];
            if (isel) { cbits = mi->ib2; abits = mi->ib; ci = idx2[i]; ai = idx1[i]; }
            int wc = oracle_bc7_weight(cbits, ci), wa = oracle_bc7_weight(abits, ai);
            for (int c = 0; c < 3; ++c) rgba[c] = interp(col[0][0][c], col[0][1][c], wc);
            rgba[3] = interp(col[0][0][3], col[0][1][3], wa);
        }
        if (rot) { int t = rgba[3]; rgba[3] = rgba[rot - 1]; rgba[rot - 1] = t; }
        for (int c = 0; c < 4; ++c) out[4 * i + c] = (uint8_t)rgba[c];
    }
    return r.pos;
}

/* Decodes a (w x h)-texel BC7 image (blocks row-major) to RGBA8. */
void oracle_bc7_decode_image(const uint8_t *blocks, int w, int h, uint8_t *rgba)
{
    int bw = w / 4, bh = h / 4;
    uint8_t tex[64];
    for (int by = 0; by < bh; ++by)
        for (int bx = 0; bx < bw; ++bx) {
            oracle_bc7_decode_block(blocks + 16 * (by * bw + bx), tex);
            for (int r = 0; r < 4; ++r)
                for (int c = 0; c < 4; ++c)
                    memcpy(rgba + 4 * ((by * 4 + r) * w + bx * 4 + c), tex + 4 * (4 * r + c), 4);
        }
}

/* ------------------------------------------------------------------ */
/* BC1 / BC4 and their combinations BC3, BC5 ("DXTC spans BC1     */
/* through BC7 ... BC5 for normal maps"; reading   */
/* R29).  D3D11 block layouts, little-endian; the interpolated palette */
/* entries use integer division (truncation), as Pillow's decoder does.*/
/* ------------------------------------------------------------------ */

/* BC1 colour block (8 bytes): c0, c1 as RGB565 (u16 LE at bytes 0, 2),
 * then 16 2-bit indices (u32 LE at byte 4, texel i = 4*row+col at bits
 * 2i).  565 -> 888 by bit replication.  c0 > c1 (or always, for the
 * colour half of BC3): palette c0, c1, (2c0+c1)/3, (c0+2c1)/3; else
 * c0, c1, (c0+c1)/2, transparent black (0,0,0,0).  A = 255 otherwise. */
void oracle_bc1_decode_block(const uint8_t blk[8], uint8_t out[64], int always_four)
{
    int c[2] = {blk[0] | (blk[1] << 8), blk[2] | (blk[3] << 8)};
    int pal[4][4];
    for (int e = 0; e < 2; ++e) {
        pal[e][0] = expand8(c[e] >> 11, 5);
        pal[e][1] = expand8((c[e] >> 5) & 63, 6);
        pal[e][2] = expand8(c[e] & 31, 5);
        pal[e][3] = 255;
    }
    int four = always_four || c[0] > c[1];
    for (int ch = 0; ch < 3; ++ch) {
        if (four) {
            pal[2][ch] = (2 * pal[0][ch] + pal[1][ch]) / 3;
            pal[3][ch] = (pal[0][ch] + 2 * pal[1][ch]) / 3;
        } else {
            pal[2][ch] = (pal[0][ch] + pal[1][ch]) / 2;
            pal[3][ch] = 0;
        }
    }
    pal[2][3] = 255;
    pal[3][3] = four ? 255 : 0;
    uint32_t idx = (uint32_t)blk[4] | ((uint32_t)blk[5] << 8) | ((uint32_t)blk[6] << 16) | ((uint32_t)blk[7] << 24);
    for (int i = 0; i < 16; ++i) {
        int q = (idx >> (2 * i)) & 3;
        for (int ch = 0; ch < 4; ++ch) out[4 * i + ch] = (uint8_t)pal[q][ch];
    }
}

/* BC4 (unsigned) block (8 bytes): a0, a1 (bytes 0, 1), then 16 3-bit
 * indices (48 bits LE from byte 2, texel i at bits 3i).  a0 > a1:
 * palette a0, a1, ((8-j) a0 + (j-1) a1) / 7 for j = 2..7; else a0, a1,
 * ((6-j) a0 + (j-1) a1) / 5 for j = 2..5, then 0 and 255.              */
void oracle_bc4_decode_block(const uint8_t blk[8], uint8_t out[16])
{
    int a0 = blk[0], a1 = blk[1], pal[8];
    pal[0] = a0;
    pal[1] = a1;
    if (a0 > a1) {
        for (int j = 2; j < 8; ++j) pal[j] = ((8 - j) * a0 + (j - 1) * a1) / 7;
    } else {
        for (int j = 2; j < 6; ++j) pal[j] = ((6 - j) * a0 + (j - 1) * a1) / 5;
        pal[6] = 0;
        pal[7] = 255;
    }
    uint64_t idx = 0;
    for (int b = 0; b < 6; ++b) idx |= (uint64_t)blk[2 + b] << (8 * b);
    for (int i = 0; i < 16; ++i) out[i] = (uint8_t)pal[(idx >> (3 * i)) & 7];
}

/* BC3 (16 bytes): a BC4 block for A, then a BC1 colour block for RGB
 * decoded in four-colour mode whatever the endpoint order.             */
void oracle_bc3_decode_block(const uint8_t blk[16], uint8_t out[64])
{
    uint8_t a[16];
    oracle_bc1_decode_block(blk + 8, out, 1);
    oracle_bc4_decode_block(blk, a);
    for (int i = 0; i < 16; ++i) out[4 * i + 3] = a[i];
}

/* BC5 (16 bytes): BC4 blocks for channel 0 (R) then channel 1 (G);
 * out = 16 texels x 2 channels.                                        */
void oracle_bc5_decode_block(const uint8_t blk[16], uint8_t out[32])
{
    uint8_t r[16], g[16];
    oracle_bc4_decode_block(blk, r);
    oracle_bc4_decode_block(blk + 8, g);
    for (int i = 0; i < 16; ++i) {
        out[2 * i] = r[i];
        out[2 * i + 1] = g[i];
    }
}

/* ------------------------------------------------------------------ */
/* Feature fetch and sampling (readings R1, R2, R4, R5, R8).    */
/* ------------------------------------------------------------------ */

/* A 2D feature map of rx x ry texels with nc channels, stored in fmt.
 * BC7 maps are always 4 channels (RGBA).                               */
typedef struct { const uint8_t *base; int fmt, rx, ry, nc; } map2d;

/* Dequantised texel value (R8: q/255 for BC7 and U8; the stored value for
 * F16).  BC7: the whole block is decoded for every fetch.             */
static double fetch(const map2d *m, int a, int b, int c)
{
    if (m->fmt == OR_FMT_BC7 || m->fmt == OR_FMT_BC1 || m->fmt == OR_FMT_BC3 || m->fmt == OR_FMT_BC5) {
        uint8_t tex[64];
        size_t bsz = m->fmt == OR_FMT_BC1 ? 8 : 16;
        const uint8_t *blk = m->base + bsz * ((b / 4) * (m->rx / 4) + (a / 4));
        if (m->fmt == OR_FMT_BC7) oracle_bc7_decode_block(blk, tex);
        else if (m->fmt == OR_FMT_BC1) oracle_bc1_decode_block(blk, tex, 0);
        else if (m->fmt == OR_FMT_BC3) oracle_bc3_decode_block(blk, tex);
        else oracle_bc5_decode_block(blk, tex);
        int nch = m->fmt == OR_FMT_BC5 ? 2 : 4;
        return tex[nch * (4 * (b % 4) + (a % 4)) + c] / 255.0;   /* R8: q/255 */
    }
    size_t k = ((size_t)b * m->rx + a) * m->nc + c;
    if (m->fmt == OR_FMT_U8) return m->base[k] / 255.0;
    uint16_t h;
    memcpy(&h, m->base + 2 * k, 2);
    return oracle_half_to_double(h);
}

static int clampi(int x, int lo, int hi) { return x < lo ? lo : (x > hi ? hi : x); }

/* Bilinear sample at normalised coordinates (a, b): texel centres at
 * (i+0.5)/R, clamp-to-edge addressing (R1).                            */
static void bilinear(const map2d *m, double a, double b, double *out)
{
    double sx = a * m->rx - 0.5, sy = b * m->ry - 0.5;
    double fx0 = floor(sx), fy0 = floor(sy);
    double fx = sx - fx0, fy = sy - fy0;
    int x0 = clampi((int)fx0, 0, m->rx - 1), x1 = clampi((int)fx0 + 1, 0, m->rx - 1);
    int y0 = clampi((int)fy0, 0, m->ry - 1), y1 = clampi((int)fy0 + 1, 0, m->ry - 1);
    for (int c = 0; c < m->nc; ++c)
        out[c] = (1 - fx) * (1 - fy) * fetch(m, x0, y0, c) + fx * (1 - fy) * fetch(m, x1, y0, c)
               + (1 - fx) * fy * fetch(m, x0, y1, c) + fx * fy * fetch(m, x1, y1, c);
}

/* exported for the sampler pins: one 2D map without tile offsets */
void oracle_sample2d(const uint8_t *base, int fmt, int rx, int ry, int nc, double a, double b, double *out)
{
    map2d m = {base, fmt, rx, ry, nc};
    bilinear(&m, a, b, out);
}

static size_t bytes_2d(int fmt, int rx, int ry, int nc)
{
    if (fmt == OR_FMT_BC7 || fmt == OR_FMT_BC3 || fmt == OR_FMT_BC5) return (size_t)(rx / 4) * (ry / 4) * 16;
    if (fmt == OR_FMT_BC1) return (size_t)(rx / 4) * (ry / 4) * 8;
    return (size_t)rx * ry * nc * (fmt == OR_FMT_U8 ? 1 : 2);
}

size_t oracle_tile_bytes_uv(const oracle_layout *L)  { return bytes_2d(L->fmt_uv, L->uv_res, L->uv_res, 4); }
size_t oracle_tile_bytes_uvt(const oracle_layout *L) { return (size_t)L->uvt_depth * bytes_2d(L->fmt_uvt, L->uvt_res, L->uvt_res, 4); }
size_t oracle_tile_bytes_line(const oracle_layout *L){ return bytes_2d(L->fmt_line, L->line_res, L->line_t, 2); }
size_t oracle_mlp_params(int h) { return (size_t)16 * h + h + (size_t)h * h + h + 3 * (size_t)h + 3; }

/* Trilinear sample of the D-deep volume (R4): s = t*D - 0.5, texel-centre
 * convention along depth, clamp, then bilinear in each slice.          */
static void trilinear_uvt(const oracle_layout *L, const uint8_t *vol, double u, double v, double t, double *out)
{
    size_t slice = bytes_2d(L->fmt_uvt, L->uvt_res, L->uvt_res, 4);
    double s = t * L->uvt_depth - 0.5;
    double k0d = floor(s), tau = s - k0d;
    int k0 = clampi((int)k0d, 0, L->uvt_depth - 1), k1 = clampi((int)k0d + 1, 0, L->uvt_depth - 1);
    map2d m0 = {vol + slice * k0, L->fmt_uvt, L->uvt_res, L->uvt_res, 4};
    map2d m1 = {vol + slice * k1, L->fmt_uvt, L->uvt_res, L->uvt_res, 4};
    double a[4], b[4];
    bilinear(&m0, u, v, a);
    bilinear(&m1, u, v, b);
    for (int c = 0; c < 4; ++c) out[c] = (1 - tau) * a[c] + tau * b[c];
}

void oracle_sample_uvt(const oracle_layout *L, const uint8_t *vol, double u, double v, double t, double *out)
{
    trilinear_uvt(L, vol, u, v, t, out);
}

/* gamma(t) = [sin(2^0 pi t), cos(2^0 pi t), sin(2^1 pi t), cos(2^1 pi t)]  (Eq. 4) */
void oracle_gamma(double t, double g[4])
{
    g[0] = sin(M_PI * t);
    g[1] = cos(M_PI * t);
    g[2] = sin(2.0 * M_PI * t);
    g[3] = cos(2.0 * M_PI * t);
}

/* Eq. 4 input vector x = [V_uvt, V_uv, V_ut, V_vt, gamma(t)] (R6) for
 * tile k at normalised (u, v) and time t.                              */
void oracle_features(const oracle_layout *L, const oracle_maps *M, int k, double u, double v, double t, double x[16])
{
    map2d uv = {M->uv + oracle_tile_bytes_uv(L) * k, L->fmt_uv, L->uv_res, L->uv_res, 4};
    map2d ut = {M->ut + oracle_tile_bytes_line(L) * k, L->fmt_line, L->line_res, L->line_t, 2};
    map2d vt = {M->vt + oracle_tile_bytes_line(L) * k, L->fmt_line, L->line_res, L->line_t, 2};
    trilinear_uvt(L, M->uvt + oracle_tile_bytes_uvt(L) * k, u, v, t, x + 0);   /* V_uvt */
    bilinear(&uv, u, v, x + 4);                                                  /* V_uv  */
    bilinear(&ut, u, t, x + 8);                                                  /* V_ut: axes (u, t) */
    bilinear(&vt, v, t, x + 10);                                                 /* V_vt: axes (v, t) */
    oracle_gamma(t, x + 12);
}

/* ------------------------------------------------------------------ */
/* Decoder MLP G_Phi: 16 -> h -> h -> 3, GELU on hidden layers, linear
 * output.  Weights f16, PyTorch [out][in] order (R11).         */
/* ------------------------------------------------------------------ */
double oracle_gelu(double z, int variant)
{
    if (variant == OR_GELU_TANH)
        return 0.5 * z * (1.0 + tanh(sqrt(2.0 / M_PI) * (z + 0.044715 * z * z * z)));
    return 0.5 * z * (1.0 + erf(z / sqrt(2.0)));
}

static void linear(const uint16_t *W, const uint16_t *b, int nout, int nin, const double *in, double *out)
{
    for (int o = 0; o < nout; ++o) {
        double acc = oracle_half_to_double(b[o]);
        for (int i = 0; i < nin; ++i) acc += oracle_half_to_double(W[o * nin + i]) * in[i];
        out[o] = acc;
    }
}

void oracle_mlp(int h, const uint16_t *w, const double x[16], int gelu, double y[3])
{
    double h1[256], h2[256];
    const uint16_t *W1 = w, *b1 = W1 + 16 * h, *W2 = b1 + h, *b2 = W2 + h * h, *W3 = b2 + h, *b3 = W3 + 3 * h;
    linear(W1, b1, h, 16, x, h1);
    for (int i = 0; i < h; ++i) h1[i] = oracle_gelu(h1[i], gelu);
    linear(W2, b2, h, h, h1, h2);
    for (int i = 0; i < h; ++i) h2[i] = oracle_gelu(h2[i], gelu);
    linear(W3, b3, 3, h, h2, y);
}

/* ------------------------------------------------------------------ */
/* Tile decode (readings R2, R3, R12, R16).               */
/* ------------------------------------------------------------------ */

/* mirror a core coordinate without repeating the edge (R3) */
static int mirror(int i, int C)
{
    if (i < 0) i = -i;
    if (i >= C) i = 2 * (C - 1) - i;
    return i;
}

/* I(u,v,t) for padded texel (x, y) of tile k -> y3 (fp64, pre-clamp) */
void oracle_texel(const oracle_layout *L, const oracle_maps *M, int k, int x, int y, double t, double out[3])
{
    int C = L->core, i = x - L->border, j = y - L->border;
    if (L->border_mode == OR_BORDER_MIRROR) { i = mirror(i, C); j = mirror(j, C); }
    double u = (i + 0.5) / C, v = (j + 0.5) / C;
    double feat[16];
    oracle_features(L, M, k, u, v, t, feat);
    oracle_mlp(L->hidden, M->mlp + oracle_mlp_params(L->hidden) * k, feat, L->gelu, out);
}

typedef struct {
    const oracle_layout *L; const oracle_maps *M; const uint32_t *ids; uint32_t n; double t;
    double *out; int full; int next_row; pthread_mutex_t *mu;
} job;

static void do_row(job *J, int row)
{
    const oracle_layout *L = J->L;
    int C = L->core, P = C + 2 * L->border;
    if (!J->full) {
        int r = row / P, y = row % P;
        int k = (int)J->ids[r];
        for (int x = 0; x < P; ++x)
            oracle_texel(L, J->M, k, x, y, J->t, J->out + 3 * (((size_t)r * P + y) * P + x));
    } else {
        /* decode_full: core texels only, atlas placement
         * tile id k = (a*tiles_y + ty)*tiles_x + tx                        */
        int k = row / C, j = row % C;
        int tx = k % L->tiles_x, ty = (k / L->tiles_x) % L->tiles_y, a = k / (L->tiles_x * L->tiles_y);
        size_t W = (size_t)L->tiles_x * C, Hh = (size_t)L->tiles_y * C;
        for (int i = 0; i < C; ++i)
            oracle_texel(L, J->M, k, i + L->border, j + L->border, J->t,
                         J->out + 3 * ((size_t)a * Hh * W + ((size_t)ty * C + j) * W + (size_t)tx * C + i));
    }
}

static void *worker(void *arg)
{
    job *J = (job *)arg;
    int C = J->L->core, P = C + 2 * J->L->border;
    int rows = J->full ? J->L->num_tiles * C : (int)J->n * P;
    for (;;) {
        pthread_mutex_lock(J->mu);
        int row = J->next_row++;
        pthread_mutex_unlock(J->mu);
        if (row >= rows) break;
        do_row(J, row);
    }
    return NULL;
}

static int run(job *J, int nthreads)
{
    pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
    J->mu = &mu;
    J->next_row = 0;
    if (nthreads <= 1) { worker(J); return 0; }
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * nthreads);
    for (int i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, worker, J);
    for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
    free(th);
    return 0;
}

static int check_ids(const oracle_layout *L, const uint32_t *ids, uint32_t n)
{
    for (uint32_t r = 0; r < n; ++r) if (ids[r] >= (uint32_t)L->num_tiles) return -1;
    return 0;
}

/* y_out: [n][P][P][3] fp64 (padded tile, mirrored border) */
int oracle_decode_tiles(const oracle_layout *L, const oracle_maps *M, const uint32_t *ids, uint32_t n,
                        double t, double *y_out, int nthreads)
{
    if (check_ids(L, ids, n)) return -1;
    job J = {L, M, ids, n, t, y_out, 0, 0, NULL};
    return run(&J, nthreads);
}

/* y_out: [atlases][tiles_y*C][tiles_x*C][3] fp64 (core texels only) */
int oracle_decode_full(const oracle_layout *L, const oracle_maps *M, double t, double *y_out, int nthreads)
{
    job J = {L, M, NULL, 0, t, y_out, 1, 0, NULL};
    return run(&J, nthreads);
}

/* Output quantisation to RGBA8 (R12): RN-even(clamp(y,0,1)*255), A = 255.
 * Two precisions so that the decision is taken in the precision of the
 * y being quantised (fp64 oracle y, or a kernel's fp32 y).             */
void oracle_quantize_rgba8_f64(const double *y3, size_t n, uint8_t *out)
{
    for (size_t i = 0; i < n; ++i) {
        for (int c = 0; c < 3; ++c) {
            double v = y3[3 * i + c];
            v = fmin(fmax(v, 0.0), 1.0);   /* NaN -> 0, as fmaxf does */
            out[4 * i + c] = (uint8_t)nearbyint(v * 255.0);
        }
        out[4 * i + 3] = 255;
    }
}

void oracle_quantize_rgba8_f32(const float *y, size_t stride, size_t n, uint8_t *out)
{
    /* the clamp is taken in fp32 (the kernel's precision); the product
     * clamp(y)*255 is exact in double, so nearbyint rounds the exact value
     * (RN-even) as R12 defines -- no intermediate fp32 rounding of the product */
    for (size_t i = 0; i < n; ++i) {
        for (int c = 0; c < 3; ++c) {
            float v = y[stride * i + c];
            v = fminf(fmaxf(v, 0.0f), 1.0f);
            out[4 * i + c] = (uint8_t)nearbyint((double)v * 255.0);
        }
        out[4 * i + 3] = 255;
    }
}

/* ------------------------------------------------------------------ */
/* Shading side of the page cache.             */
/*                                                                      */
/* The physical texture (page cache) holds the decoder output y in the  */
/* 8-bit 4-channel format per padded tile slot; during shading  */
/* "we first sample the page table to locate each tile within the       */
/* physical texture, then sample the physical texture",  */
/* with filtering served by the tile's border, and the per-     */
/* channel means stored at each bake time "are later used during        */
/* rendering to restore the original lightmap data" after the   */
/* gamma correction applied before training.  Readings R21-R25  */
/* (DESIGN.md): restore x^g * mu_hat(t,c) after filtering (R21), mu_hat */
/* linear between bracketing bake times (R22, SPEC postprocess),        */
/* page-table entry = (slot, time bucket) (R24), sample position and    */
/* owning tile (R25).                                                   */
/* ------------------------------------------------------------------ */

/* R22: per-channel mean at time t, linear between the bracketing bake
 * times times[0] < ... < times[n-1]; t outside [times[0], times[n-1]]
 * is an error (returns 1). */
int oracle_mean_at(const double *times, const double *means, int n, double t, double out[3])
{
    if (n < 1 || !(t >= times[0]) || !(t <= times[n - 1])) return 1;
    if (n == 1) {
        for (int c = 0; c < 3; ++c) out[c] = means[c];
        return 0;
    }
    int i = 0;
    while (i < n - 2 && t > times[i + 1]) ++i;      /* times[i] <= t <= times[i+1] */
    double lam = (t - times[i]) / (times[i + 1] - times[i]);
    for (int c = 0; c < 3; ++c) out[c] = (1.0 - lam) * means[3 * i + c] + lam * means[3 * (i + 1) + c];
    return 0;
}

/* R21/R23: undo the gamma correction and the mean normalisation */
double oracle_restore(double x, double g, double mu) { return pow(x, g) * mu; }

/* R25: one shading sample at (u, v) in [0,1]^2 of atlas `atlas`.
 * cache: [slots][P][P][4] u8 (P = C + 2B), pt: [tiles][2] int32 = (slot,
 * bucket), tile id = (atlas * tiles_y + ty) * tiles_x + tx.  The texel
 * grid of the atlas has centres at ((i + 0.5)/W, (j + 0.5)/H); the owning
 * tile is the one whose core contains the sample point; the bilinear taps
 * (at most one texel outside the core) come from that tile's slot, its
 * border supplying the outside taps.  Returns 0, or 1 when the tile is
 * not resident for `bucket` (out untouched). */
int oracle_sample_lighting(const uint8_t *cache, const int32_t *pt, int C, int B, int tiles_x, int tiles_y,
                           int atlas, double u, double v, int bucket, double g, const double mu[3], double out[3])
{
    const int P = C + 2 * B;
    const int W = tiles_x * C, H = tiles_y * C;
    u = fmin(fmax(u, 0.0), 1.0);
    v = fmin(fmax(v, 0.0), 1.0);
    int tx = (int)floor(u * tiles_x), ty = (int)floor(v * tiles_y);
    if (tx > tiles_x - 1) tx = tiles_x - 1;
    if (ty > tiles_y - 1) ty = tiles_y - 1;
    const long id = ((long)atlas * tiles_y + ty) * tiles_x + tx;
    const int slot = pt[2 * id], b = pt[2 * id + 1];
    if (slot < 0 || b != bucket) return 1;
    const double lx = u * W - 0.5 - (double)tx * C;   /* in [-0.5, C - 0.5] */
    const double ly = v * H - 0.5 - (double)ty * C;
    const double x0 = floor(lx), y0 = floor(ly);
    const double fx = lx - x0, fy = ly - y0;
    const uint8_t *s = cache + (size_t)slot * P * P * 4;
    for (int c = 0; c < 3; ++c) {
        double q[2][2];
        for (int dy = 0; dy < 2; ++dy)
            for (int dx = 0; dx < 2; ++dx) {
                const int px = (int)x0 + dx + B, py = (int)y0 + dy + B;
                q[dy][dx] = s[((size_t)py * P + px) * 4 + c] / 255.0;
            }
        const double val = (1 - fx) * (1 - fy) * q[0][0] + fx * (1 - fy) * q[0][1] + (1 - fx) * fy * q[1][0] +
                           fx * fy * q[1][1];
        out[c] = oracle_restore(val, g, mu[c]);
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* BC7 mode-6 encoder ("after training,  */
/* we not only quantize them to 8-bit, but also apply the BC7          */
/* compression algorithm", "followed by quantization and BC7     */
/* compression"; SPEC S:371-385 principal-axis endpoints + nearest     */
/* indices).  Reading R26 makes it exact integer          */
/* arithmetic, so the GPU encoder must match it bit for bit:           */
/*   1. 16*cov = 16*sum(p p^T) - sum(p) sum(p)^T (int64, exact);       */
/*   2. principal axis by 4 power iterations from the column of the     */
/*      largest-variance channel, each step w = M v then v = w with     */
/*      magnitudes shifted right until max|v| < 2^20 (sign kept);       */
/*   3. endpoints = the texels with the smallest / largest projection   */
/*      p.v (first index on ties), each quantised to 7 bits + p-bit:    */
/*      q = clamp((e - p + 1) >> 1, 0, 127) per channel, value 2q + p,  */
/*      p in {0, 1} minimising the squared error (p = 0 on ties);       */
/*   4. per texel the 4-bit index minimising the squared error of the   */
/*      decoder's own interpolation (smallest index on ties);           */
/*   5. if texel 0's index has its MSB set (mode 6 anchor), swap the    */
/*      endpoints and replace every index w by 15 - w (W4 is symmetric, */
/*      so the decoded block is unchanged);                             */
/*   6. pack LSB-first: mode 6 (0x40), R0 R1 G0 G1 B0 B1 A0 A1 (7 b),  */
/*      P0, P1, texel 0 index (3 b), texels 1..15 (4 b).                */
/* ------------------------------------------------------------------ */
static int bitlen64(uint64_t x) { int n = 0; while (x) { ++n; x >>= 1; } return n; }

static int64_t floor_div64(int64_t x, int64_t y)   /* y > 0 */
{
    int64_t q = x / y;
    if ((x % y != 0) && (x < 0)) q -= 1;
    return q;
}

static void quant_endpoint_m6(const int e[4], int val[4], int *pbit)
{
    int best = -1;
    for (int p = 0; p < 2; ++p) {
        int v[4], err = 0;
        for (int c = 0; c < 4; ++c) {
            int q = (e[c] - p + 1) >> 1;
            if (q < 0) q = 0;
            if (q > 127) q = 127;
            v[c] = 2 * q + p;
            err += (v[c] - e[c]) * (v[c] - e[c]);
        }
        if (best < 0 || err < best) {
            best = err;
            *pbit = p;
            for (int c = 0; c < 4; ++c) val[c] = v[c];
        }
    }
}

typedef struct { uint8_t *b; int pos; } bitwriter;
static void put(bitwriter *w, int v, int n)
{
    for (int i = 0; i < n; ++i) {
        if ((v >> i) & 1) w->b[w->pos >> 3] |= (uint8_t)(1u << (w->pos & 7));
        w->pos++;
    }
}

void oracle_bc7_encode_mode6(const uint8_t px[64], uint8_t out[16])
{
    int64_t S[4] = {0, 0, 0, 0}, Q[4][4];
    memset(Q, 0, sizeof(Q));
    for (int i = 0; i < 16; ++i)
        for (int c = 0; c < 4; ++c) {
            S[c] += px[4 * i + c];
            for (int d = 0; d < 4; ++d) Q[c][d] += (int64_t)px[4 * i + c] * px[4 * i + d];
        }
    int64_t M[4][4];
    for (int c = 0; c < 4; ++c)
        for (int d = 0; d < 4; ++d) M[c][d] = 16 * Q[c][d] - S[c] * S[d];
    /* step 2 */
    int cs = 0;
    for (int c = 1; c < 4; ++c)
        if (M[c][c] > M[cs][cs]) cs = c;
    int64_t v[4];
    for (int c = 0; c < 4; ++c) v[c] = M[c][cs];
    for (int it = 0; it <= 4; ++it) {
        int64_t w[4];
        if (it == 0) {
            for (int c = 0; c < 4; ++c) w[c] = v[c];
        } else {
            for (int c = 0; c < 4; ++c) {
                w[c] = 0;
                for (int d = 0; d < 4; ++d) w[c] += M[c][d] * v[d];
            }
        }
        uint64_t mx = 0;
        for (int c = 0; c < 4; ++c) {
            uint64_t a = (uint64_t)(w[c] < 0 ? -w[c] : w[c]);
            if (a > mx) mx = a;
        }
        if (mx == 0) {   /* constant block or v in the null space: keep v (or (1,1,1,1)) */
            if (it == 0) for (int c = 0; c < 4; ++c) v[c] = 1;
            break;
        }
        const int s = bitlen64(mx) > 20 ? bitlen64(mx) - 20 : 0;
        for (int c = 0; c < 4; ++c) {
            const uint64_t a = (uint64_t)(w[c] < 0 ? -w[c] : w[c]) >> s;
            v[c] = w[c] < 0 ? -(int64_t)a : (int64_t)a;
        }
    }
    /* step 3 */
    int imin = 0, imax = 0;
    int64_t dmin = 0, dmax = 0;
    for (int i = 0; i < 16; ++i) {
        int64_t d = 0;
        for (int c = 0; c < 4; ++c) d += (int64_t)px[4 * i + c] * v[c];
        if (i == 0 || d < dmin) { dmin = d; imin = i; }
        if (i == 0 || d > dmax) { dmax = d; imax = i; }
    }
    int e0[4], e1[4], E0[4], E1[4], p0, p1;
    for (int c = 0; c < 4; ++c) { e0[c] = px[4 * imin + c]; e1[c] = px[4 * imax + c]; }
    quant_endpoint_m6(e0, E0, &p0);
    quant_endpoint_m6(e1, E1, &p1);
    /* step 4 */
    int idx[16];
    for (int i = 0; i < 16; ++i) {
        int best = -1;
        for (int w = 0; w < 16; ++w) {
            int err = 0;
            for (int c = 0; c < 4; ++c) {
                const int d = interp(E0[c], E1[c], BC7_W4[w]) - px[4 * i + c];
                err += d * d;
            }
            if (best < 0 || err < best) { best = err; idx[i] = w; }
        }
    }
    /* step 4b (R26): one least-squares refit of the endpoints for these
     * indices, in exact integers -- per channel, with a = 64 - W4[idx],
     * b = W4[idx]: [S aa, S ab; S ab, S bb] (e0, e1) = 64 (S a p, S b p),
     * e = floor((2 num + det) / (2 det)) clamped to [0, 255], requantised
     * (p-bits as in step 3) and re-indexed (step 4); kept only if the total
     * squared error is strictly smaller. */
    {
        int64_t saa = 0, sab = 0, sbb = 0;
        for (int i = 0; i < 16; ++i) {
            const int64_t a = 64 - BC7_W4[idx[i]], b = BC7_W4[idx[i]];
            saa += a * a; sab += a * b; sbb += b * b;
        }
        const int64_t det = saa * sbb - sab * sab;
        if (det > 0) {
            int f0[4], f1[4], F0[4], F1[4], q0, q1, jdx[16];
            for (int c = 0; c < 4; ++c) {
                int64_t r0 = 0, r1 = 0;
                for (int i = 0; i < 16; ++i) {
                    r0 += (int64_t)(64 - BC7_W4[idx[i]]) * px[4 * i + c] * 64;
                    r1 += (int64_t)BC7_W4[idx[i]] * px[4 * i + c] * 64;
                }
                const int64_t n0 = sbb * r0 - sab * r1, n1 = saa * r1 - sab * r0;
                int64_t e0 = floor_div64(2 * n0 + det, 2 * det), e1 = floor_div64(2 * n1 + det, 2 * det);
                f0[c] = (int)(e0 < 0 ? 0 : (e0 > 255 ? 255 : e0));
                f1[c] = (int)(e1 < 0 ? 0 : (e1 > 255 ? 255 : e1));
            }
            quant_endpoint_m6(f0, F0, &q0);
            quant_endpoint_m6(f1, F1, &q1);
            int64_t err_old = 0, err_new = 0;
            for (int i = 0; i < 16; ++i) {
                int best = -1;
                for (int w = 0; w < 16; ++w) {
                    int err = 0;
                    for (int c = 0; c < 4; ++c) {
                        const int d = interp(F0[c], F1[c], BC7_W4[w]) - px[4 * i + c];
                        err += d * d;
                    }
                    if (best < 0 || err < best) { best = err; jdx[i] = w; }
                }
                err_new += best;
                for (int c = 0; c < 4; ++c) {
                    const int d = interp(E0[c], E1[c], BC7_W4[idx[i]]) - px[4 * i + c];
                    err_old += d * d;
                }
            }
            if (err_new < err_old) {
                for (int c = 0; c < 4; ++c) { E0[c] = F0[c]; E1[c] = F1[c]; }
                p0 = q0;
                p1 = q1;
                for (int i = 0; i < 16; ++i) idx[i] = jdx[i];
            }
        }
    }
    /* step 5 */
    if (idx[0] >= 8) {
        for (int c = 0; c < 4; ++c) { int t = E0[c]; E0[c] = E1[c]; E1[c] = t; }
        int t = p0; p0 = p1; p1 = t;
        for (int i = 0; i < 16; ++i) idx[i] = 15 - idx[i];
    }
    /* step 6 */
    memset(out, 0, 16);
    bitwriter bw = {out, 0};
    put(&bw, 1 << 6, 7);
    for (int c = 0; c < 4; ++c) { put(&bw, E0[c] >> 1, 7); put(&bw, E1[c] >> 1, 7); }
    put(&bw, p0, 1);
    put(&bw, p1, 1);
    put(&bw, idx[0], 3);
    for (int i = 1; i < 16; ++i) put(&bw, idx[i], 4);
}

void oracle_bc7_encode_image_mode6(const uint8_t *rgba, int w, int h, uint8_t *blocks)
{
    for (int by = 0; by < h / 4; ++by)
        for (int bx = 0; bx < w / 4; ++bx) {
            uint8_t px[64];
            for (int i = 0; i < 16; ++i)
                memcpy(px + 4 * i, rgba + ((size_t)(4 * by + i / 4) * w + 4 * bx + i % 4) * 4, 4);
            oracle_bc7_encode_mode6(px, blocks + ((size_t)by * (w / 4) + bx) * 16);
        }
}

/* ------------------------------------------------------------------ */
/* Fine-tuning step of G_Phi on frozen features (SURVEY.md §8(f) NEXT  */
/* 4, the last stage of the paper's training: "In the final training   */
/* stage, we freeze the feature maps and fine-tune the MLP under       */
/* simulated quantization and BC compression" -- here the features are */
/* the real quantized / BC7 maps -- "We use the Adam optimizer ... and  */
/* use L2 loss", GELU on the hidden layers).  Reading R27: the   */
/* loss of a tile is the mean over samples and RGB channels of the     */
/* squared error; parameters are the fp64 master copy theta in the      */
/* layout of the f16 MLP blob [W1 | b1 | W2 | b2 | W3 | b3]; Adam with  */
/* bias correction, PyTorch's update order.                            */
/* ------------------------------------------------------------------ */
static double gelu_grad(double z, int variant)
{
    if (variant == OR_GELU_TANH) {
        const double k = 0.7978845608028654, a = 0.044715;
        const double u = k * (z + a * z * z * z), th = tanh(u);
        return 0.5 * (1.0 + th) + 0.5 * z * (1.0 - th * th) * k * (1.0 + 3.0 * a * z * z);
    }
    return 0.5 * (1.0 + erf(z * 0.7071067811865476)) + z * exp(-0.5 * z * z) * 0.3989422804014327;
}

/* loss and dloss/dtheta of one tile k over S samples (u, v, t) with targets */
double oracle_train_grad(const oracle_layout *L, const oracle_maps *M, int k, const double *theta, const double *uvt,
                         const double *target, int S, double *grad)
{
    const int h = L->hidden, P = (int)oracle_mlp_params(h);
    const double *W1 = theta, *b1 = W1 + 16 * h, *W2 = b1 + h, *b2 = W2 + h * h, *W3 = b2 + h, *b3 = W3 + 3 * h;
    double *gW1 = grad, *gb1 = gW1 + 16 * h, *gW2 = gb1 + h, *gb2 = gW2 + h * h, *gW3 = gb2 + h, *gb3 = gW3 + 3 * h;
    memset(grad, 0, sizeof(double) * P);
    double loss = 0.0;
    double x[16], z1[256], g1[256], z2[256], g2[256], y[3], dy[3], dg2[256], dz2[256], dg1[256], dz1[256];
    for (int s = 0; s < S; ++s) {
        oracle_features(L, M, k, uvt[3 * s], uvt[3 * s + 1], uvt[3 * s + 2], x);
        for (int o = 0; o < h; ++o) {
            double a = b1[o];
            for (int i = 0; i < 16; ++i) a += W1[o * 16 + i] * x[i];
            z1[o] = a;
            g1[o] = oracle_gelu(a, L->gelu);
        }
        for (int o = 0; o < h; ++o) {
            double a = b2[o];
            for (int i = 0; i < h; ++i) a += W2[o * h + i] * g1[i];
            z2[o] = a;
            g2[o] = oracle_gelu(a, L->gelu);
        }
        for (int o = 0; o < 3; ++o) {
            double a = b3[o];
            for (int i = 0; i < h; ++i) a += W3[o * h + i] * g2[i];
            y[o] = a;
            const double d = y[o] - target[3 * s + o];
            loss += d * d;
            dy[o] = 2.0 * d / (3.0 * S);
        }
        for (int o = 0; o < 3; ++o) {
            gb3[o] += dy[o];
            for (int i = 0; i < h; ++i) gW3[o * h + i] += dy[o] * g2[i];
        }
        for (int i = 0; i < h; ++i) {
            double a = 0.0;
            for (int o = 0; o < 3; ++o) a += W3[o * h + i] * dy[o];
            dg2[i] = a;
            dz2[i] = a * gelu_grad(z2[i], L->gelu);
        }
        for (int o = 0; o < h; ++o) {
            gb2[o] += dz2[o];
            for (int i = 0; i < h; ++i) gW2[o * h + i] += dz2[o] * g1[i];
        }
        for (int i = 0; i < h; ++i) {
            double a = 0.0;
            for (int o = 0; o < h; ++o) a += W2[o * h + i] * dz2[o];
            dg1[i] = a;
            dz1[i] = a * gelu_grad(z1[i], L->gelu);
        }
        for (int o = 0; o < h; ++o) {
            gb1[o] += dz1[o];
            for (int i = 0; i < 16; ++i) gW1[o * 16 + i] += dz1[o] * x[i];
        }
    }
    return loss / (3.0 * S);
}

/* one Adam step (PyTorch order): m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2;
 * theta -= lr * (m / (1 - b1^step)) / (sqrt(v / (1 - b2^step)) + eps) */
void oracle_adam(double *theta, double *m, double *v, const double *g, int P, int step, double lr, double b1,
                 double b2, double eps)
{
    const double c1 = 1.0 - pow(b1, step), c2 = 1.0 - pow(b2, step);
    for (int i = 0; i < P; ++i) {
        m[i] = b1 * m[i] + (1.0 - b1) * g[i];
        v[i] = b2 * v[i] + (1.0 - b2) * g[i] * g[i];
        theta[i] -= lr * (m[i] / c1) / (sqrt(v[i] / c2) + eps);
    }
}

/* ------------------------------------------------------------------ */
/* Full training step: BC-simulated feature   */
/* maps (Eq. 6-7: "we divide each feature map into 4x4      */
/* blocks, where the feature values within each block are represented  */
/* by a set of endpoints E and weights W ... f_p = (1 - w_p) e1 +       */
/* w_p e2"), uniform noise on the sampled vectors (Eq. 5:    */
/* alpha = 1/256; "Noise is then added to the sampled vector     */
/* V_uvt, V_uv"), plain line grids, the per-tile MLP, L2 loss, Adam.   */
/* Reading R28: parameters of one tile, fp64 here, in the   */
/* order [MLP blob | F_uv blocks | F_uvt slices' blocks | F_ut | F_vt],  */
/* each block [e1 RGBA | e2 RGBA | w_0..w_15]; the noise draws are      */
/* inputs (n[12] per sample, in [-0.5, 0.5)); after each Adam step the  */
/* BC endpoints / weights and the line grids are projected onto [0,1].  */
/* ------------------------------------------------------------------ */
typedef struct {
    size_t mlp, uv, uvt, ut, vt, total;
} full_offsets;

static full_offsets full_layout(const oracle_layout *L)
{
    full_offsets o;
    o.mlp = 0;
    o.uv = oracle_mlp_params(L->hidden);
    o.uvt = o.uv + (size_t)(L->uv_res / 4) * (L->uv_res / 4) * 24;
    o.ut = o.uvt + (size_t)L->uvt_depth * (L->uvt_res / 4) * (L->uvt_res / 4) * 24;
    o.vt = o.ut + (size_t)L->line_t * L->line_res * 2;
    o.total = o.vt + (size_t)L->line_t * L->line_res * 2;
    return o;
}

size_t oracle_train_full_params(const oracle_layout *L) { return full_layout(L).total; }

/* a differentiable 2D map: BC-simulated (blocks) or plain (grid) */
typedef struct {
    const double *p;   /* parameters */
    double *g;         /* their gradient (or NULL) */
    int bc, rx, ry, nc;
} dmap;

static double dfetch(const dmap *m, int a, int b, int c)
{
    if (m->bc) {
        const double *blk = m->p + ((size_t)(b / 4) * (m->rx / 4) + a / 4) * 24;
        const double w = blk[8 + 4 * (b % 4) + (a % 4)];
        return (1.0 - w) * blk[c] + w * blk[4 + c];    /* Eq. 7 */
    }
    return m->p[((size_t)b * m->rx + a) * m->nc + c];
}

static void dscatter(const dmap *m, int a, int b, int c, double gv)
{
    if (m->bc) {
        const size_t base = ((size_t)(b / 4) * (m->rx / 4) + a / 4) * 24;
        const double *blk = m->p + base;
        const int pi = 4 * (b % 4) + (a % 4);
        const double w = blk[8 + pi];
        m->g[base + c] += gv * (1.0 - w);
        m->g[base + 4 + c] += gv * w;
        m->g[base + 8 + pi] += gv * (blk[4 + c] - blk[c]);
        return;
    }
    m->g[((size_t)b * m->rx + a) * m->nc + c] += gv;
}

/* bilinear (R1) forward, or backward with upstream gradient gout[nc] */
static void dbilinear(const dmap *m, double a, double b, double *out, const double *gout)
{
    double sx = a * m->rx - 0.5, sy = b * m->ry - 0.5;
    double fx0 = floor(sx), fy0 = floor(sy);
    double fx = sx - fx0, fy = sy - fy0;
    int x0 = clampi((int)fx0, 0, m->rx - 1), x1 = clampi((int)fx0 + 1, 0, m->rx - 1);
    int y0 = clampi((int)fy0, 0, m->ry - 1), y1 = clampi((int)fy0 + 1, 0, m->ry - 1);
    const double w00 = (1 - fx) * (1 - fy), w10 = fx * (1 - fy), w01 = (1 - fx) * fy, w11 = fx * fy;
    for (int c = 0; c < m->nc; ++c) {
        if (gout) {
            dscatter(m, x0, y0, c, w00 * gout[c]);
            dscatter(m, x1, y0, c, w10 * gout[c]);
            dscatter(m, x0, y1, c, w01 * gout[c]);
            dscatter(m, x1, y1, c, w11 * gout[c]);
        } else {
            out[c] = w00 * dfetch(m, x0, y0, c) + w10 * dfetch(m, x1, y0, c) + w01 * dfetch(m, x0, y1, c)
                   + w11 * dfetch(m, x1, y1, c);
        }
    }
}

/* features x[16] of one sample (forward) or their gradient scatter (backward, gx[12]) */
static void full_features(const oracle_layout *L, const double *theta, double *grad, double u, double v, double t,
                          const double *noise, double *x, const double *gx)
{
    const full_offsets o = full_layout(L);
    const double alpha = 1.0 / 256.0;
    const size_t slice = (size_t)(L->uvt_res / 4) * (L->uvt_res / 4) * 24;
    double s = t * L->uvt_depth - 0.5, k0d = floor(s), tau = s - k0d;
    int k0 = clampi((int)k0d, 0, L->uvt_depth - 1), k1 = clampi((int)k0d + 1, 0, L->uvt_depth - 1);
    dmap m0 = {theta + o.uvt + slice * k0, grad ? grad + o.uvt + slice * k0 : NULL, 1, L->uvt_res, L->uvt_res, 4};
    dmap m1 = {theta + o.uvt + slice * k1, grad ? grad + o.uvt + slice * k1 : NULL, 1, L->uvt_res, L->uvt_res, 4};
    dmap muv = {theta + o.uv, grad ? grad + o.uv : NULL, 1, L->uv_res, L->uv_res, 4};
    dmap mut = {theta + o.ut, grad ? grad + o.ut : NULL, 0, L->line_res, L->line_t, 2};
    dmap mvt = {theta + o.vt, grad ? grad + o.vt : NULL, 0, L->line_res, L->line_t, 2};
    if (gx) {
        double g0[4], g1[4];
        for (int c = 0; c < 4; ++c) { g0[c] = (1 - tau) * gx[c]; g1[c] = tau * gx[c]; }
        dbilinear(&m0, u, v, NULL, g0);
        dbilinear(&m1, u, v, NULL, g1);
        dbilinear(&muv, u, v, NULL, gx + 4);
        dbilinear(&mut, u, t, NULL, gx + 8);
        dbilinear(&mvt, v, t, NULL, gx + 10);
        return;
    }
    double a[4], b[4];
    dbilinear(&m0, u, v, a, NULL);
    dbilinear(&m1, u, v, b, NULL);
    for (int c = 0; c < 4; ++c) x[c] = (1 - tau) * a[c] + tau * b[c];
    dbilinear(&muv, u, v, x + 4, NULL);
    dbilinear(&mut, u, t, x + 8, NULL);
    dbilinear(&mvt, v, t, x + 10, NULL);
    for (int i = 0; i < 12; ++i) x[i] += alpha * noise[i];   /* Eq. 5 */
    oracle_gamma(t, x + 12);
}

/* loss and gradient over the whole parameter vector of one tile */
double oracle_train_full_grad(const oracle_layout *L, const double *theta, const double *uvt, const double *target,
                              const double *noise, int S, double *grad)
{
    const int h = L->hidden;
    const full_offsets o = full_layout(L);
    const double *W1 = theta, *b1 = W1 + 16 * h, *W2 = b1 + h, *b2 = W2 + h * h, *W3 = b2 + h, *b3 = W3 + 3 * h;
    double *gW1 = grad, *gb1 = gW1 + 16 * h, *gW2 = gb1 + h, *gb2 = gW2 + h * h, *gW3 = gb2 + h, *gb3 = gW3 + 3 * h;
    memset(grad, 0, sizeof(double) * o.total);
    double loss = 0.0;
    double x[16], z1[256], g1[256], z2[256], g2[256], dy[3], dz2[256], dz1[256], gx[12];
    for (int s = 0; s < S; ++s) {
        full_features(L, theta, NULL, uvt[3 * s], uvt[3 * s + 1], uvt[3 * s + 2], noise + 12 * s, x, NULL);
        for (int oo = 0; oo < h; ++oo) {
            double a = b1[oo];
            for (int i = 0; i < 16; ++i) a += W1[oo * 16 + i] * x[i];
            z1[oo] = a;
            g1[oo] = oracle_gelu(a, L->gelu);
        }
        for (int oo = 0; oo < h; ++oo) {
            double a = b2[oo];
            for (int i = 0; i < h; ++i) a += W2[oo * h + i] * g1[i];
            z2[oo] = a;
            g2[oo] = oracle_gelu(a, L->gelu);
        }
        for (int oo = 0; oo < 3; ++oo) {
            double a = b3[oo];
            for (int i = 0; i < h; ++i) a += W3[oo * h + i] * g2[i];
            const double d = a - target[3 * s + oo];
            loss += d * d;
            dy[oo] = 2.0 * d / (3.0 * S);
        }
        for (int oo = 0; oo < 3; ++oo) {
            gb3[oo] += dy[oo];
            for (int i = 0; i < h; ++i) gW3[oo * h + i] += dy[oo] * g2[i];
        }
        for (int i = 0; i < h; ++i) {
            double a = 0.0;
            for (int oo = 0; oo < 3; ++oo) a += W3[oo * h + i] * dy[oo];
            dz2[i] = a * gelu_grad(z2[i], L->gelu);
        }
        for (int oo = 0; oo < h; ++oo) {
            gb2[oo] += dz2[oo];
            for (int i = 0; i < h; ++i) gW2[oo * h + i] += dz2[oo] * g1[i];
        }
        for (int i = 0; i < h; ++i) {
            double a = 0.0;
            for (int oo = 0; oo < h; ++oo) a += W2[oo * h + i] * dz2[oo];
            dz1[i] = a * gelu_grad(z1[i], L->gelu);
        }
        for (int oo = 0; oo < h; ++oo) {
            gb1[oo] += dz1[oo];
            for (int i = 0; i < 16; ++i) gW1[oo * 16 + i] += dz1[oo] * x[i];
        }
        for (int i = 0; i < 12; ++i) {
            double a = 0.0;
            for (int oo = 0; oo < h; ++oo) a += W1[oo * 16 + i] * dz1[oo];
            gx[i] = a;
        }
        full_features(L, theta, grad, uvt[3 * s], uvt[3 * s + 1], uvt[3 * s + 2], noise + 12 * s, NULL, gx);
    }
    return loss / (3.0 * S);
}

/* R28 projection after an Adam step: BC endpoints / weights and line grids onto [0,1] */
void oracle_train_full_project(const oracle_layout *L, double *theta)
{
    const full_offsets o = full_layout(L);
    for (size_t i = o.uv; i < o.total; ++i) theta[i] = fmin(fmax(theta[i], 0.0), 1.0);
}

/* ------------------------------------------------------------------ */
/* Export of fully trained tiles to a deployable Theta (SURVEY.md 8(f) */
/* NEXT 3 "u8 PTQ plus a BC7 encoder", "BC compression on the    */
/* final generated feature maps"; reading R30).                 */
/* Per tile, from its fp32 parameter vector (R28 layout):              */
/*  * F_uv and every F_uvt slice: each block's 16 texels by Eq. 7 in   */
/*    fp32, x = (1 - w) e1 + w e2 (every operation rounded to fp32, no */
/*    fused multiply-add: the trainer's precision, so the integer      */
/*    decision below is taken in it), post-training quantisation       */
/*    q = RN-even(clamp(x, 0, 1) * 255), then BC7 mode 6 (R26);        */
/*  * F_ut, F_vt: q = RN-even(clamp(v, 0, 1) * 255), u8 [T][U][2];     */
/*  * the MLP: fp32 -> f16, RN-even.                                   */
/* Outputs in ndgi_load's dense per-tile layouts (BC7, BC7, U8, f16).  */
/* ------------------------------------------------------------------ */
uint8_t oracle_ptq_u8(float x)
{
    x = x < 0.0f ? 0.0f : (x > 1.0f ? 1.0f : x);
    float s = x * 255.0f;
    return (uint8_t)rintf(s);
}

/* IEEE binary16 of a float, round to nearest even */
uint16_t oracle_float_to_half(float f)
{
    uint32_t x;
    memcpy(&x, &f, 4);
    uint32_t sign = (x >> 16) & 0x8000u, ax = x & 0x7fffffffu;
    if (ax >= 0x7f800000u) return (uint16_t)(sign | 0x7c00u | (ax > 0x7f800000u ? 0x200u : 0u));
    if (ax >= 0x477ff000u) return (uint16_t)(sign | 0x7c00u);            /* >= 65520: inf */
    if (ax < 0x38800000u) {                                                /* < 2^-14: subnormal */
        double r = nearbyint((double)fabsf(f) * 16777216.0);               /* units of 2^-24 */
        return (uint16_t)(sign | (uint32_t)r);
    }
    uint32_t h = ((((ax >> 23) - 127u + 15u)) << 10) | ((ax & 0x7fffffu) >> 13);
    uint32_t rem = ax & 0x1fffu;
    if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) h++;
    return (uint16_t)(sign | h);
}

static void bc_map_image(const float *blocks, int R, uint8_t *rgba)
{
    int nb = R / 4;
    for (int by = 0; by < nb; ++by)
        for (int bx = 0; bx < nb; ++bx) {
            const float *blk = blocks + ((size_t)by * nb + bx) * 24;
            for (int p = 0; p < 16; ++p) {
                float w = blk[8 + p];
                for (int c = 0; c < 4; ++c) {
                    float a = 1.0f - w;
                    float t1 = a * blk[c];
                    float t2 = w * blk[4 + c];
                    float x = t1 + t2;                                      /* Eq. 7 */
                    rgba[((size_t)(4 * by + p / 4) * R + 4 * bx + p % 4) * 4 + c] = oracle_ptq_u8(x);
                }
            }
        }
}

void oracle_train_full_export(const oracle_layout *L, const float *theta, uint8_t *uv, uint8_t *uvt, uint8_t *ut,
                              uint8_t *vt, uint16_t *mlp)
{
    const full_offsets o = full_layout(L);
    const int R = L->uv_res, R3 = L->uvt_res, D = L->uvt_depth;
    const size_t uvb = (size_t)(R / 4) * (R / 4) * 16, uvtb = (size_t)(R3 / 4) * (R3 / 4) * 16;
    const size_t nl = (size_t)L->line_t * L->line_res * 2, pm = oracle_mlp_params(L->hidden);
    uint8_t *img = (uint8_t *)malloc((size_t)(R > R3 ? R : R3) * (R > R3 ? R : R3) * 4);
    for (int k = 0; k < L->num_tiles; ++k) {
        const float *th = theta + (size_t)k * o.total;
        bc_map_image(th + o.uv, R, img);
        oracle_bc7_encode_image_mode6(img, R, R, uv + k * uvb);
        for (int d = 0; d < D; ++d) {
            bc_map_image(th + o.uvt + (size_t)d * (R3 / 4) * (R3 / 4) * 24, R3, img);
            oracle_bc7_encode_image_mode6(img, R3, R3, uvt + ((size_t)k * D + d) * uvtb);
        }
        for (size_t i = 0; i < nl; ++i) {
            ut[k * nl + i] = oracle_ptq_u8(th[o.ut + i]);
            vt[k * nl + i] = oracle_ptq_u8(th[o.vt + i]);
        }
        for (size_t i = 0; i < pm; ++i) mlp[k * pm + i] = oracle_float_to_half(th[i]);
    }
    free(img);
}

/* ------------------------------------------------------------------ */
/* BC7 multi-mode search (SURVEY.md 8(f) NEXT 3 "first mode 6 ... then */
/* multi-mode search"; reading R31).  Candidates in this order, */
/* each scored by the squared error of its DECODED block (the pinned   */
/* decoder above) against the input; a later candidate replaces the    */
/* best only if strictly better:                                        */
/*  1. mode 6 (R26);                                                    */
/*  2. mode 5, rotation r = 0..3 (A swapped with R, G, B for r = 1..3): */
/*     RGB endpoints = the texels extreme along the integer principal   */
/*     axis of RGB, 7-bit codes (nearest after bit replication, ties to */
/*     the lower code); alpha endpoints = min / max alpha (8 bits);     */
/*     2-bit colour and alpha indices (nearest, ties to the lower       */
/*     index); anchor fix per index set;                                */
/*  3. mode 7, partition p = 0..63: per subset, RGBA endpoints = the    */
/*     subset's texels extreme along its principal axis, 5-bit codes +  */
/*     one p-bit per endpoint (the p-bit with the smaller squared       */
/*     endpoint error, ties to 0), 2-bit indices, anchor fix per        */
/*     subset.                                                          */
/* The principal axis is R26 step 2 over the chosen texels / channels.  */
/* ------------------------------------------------------------------ */
static void axis_extremes(const uint8_t px[64], uint32_t mask, const int *chs, int nc, int *imin, int *imax)
{
    int64_t S[4] = {0, 0, 0, 0}, Q[4][4], M[4][4], v[4];
    memset(Q, 0, sizeof(Q));
    int n = 0;
    for (int i = 0; i < 16; ++i) {
        if (!((mask >> i) & 1u)) continue;
        n++;
        for (int c = 0; c < nc; ++c) {
            S[c] += px[4 * i + chs[c]];
            for (int d = 0; d < nc; ++d) Q[c][d] += (int64_t)px[4 * i + chs[c]] * px[4 * i + chs[d]];
        }
    }
    for (int c = 0; c < nc; ++c)
        for (int d = 0; d < nc; ++d) M[c][d] = n * Q[c][d] - S[c] * S[d];
    int cs = 0;
    for (int c = 1; c < nc; ++c)
        if (M[c][c] > M[cs][cs]) cs = c;
    for (int c = 0; c < nc; ++c) v[c] = M[c][cs];
    for (int it = 0; it <= 4; ++it) {
        int64_t w[4];
        for (int c = 0; c < nc; ++c) {
            if (it == 0) { w[c] = v[c]; continue; }
            w[c] = 0;
            for (int d = 0; d < nc; ++d) w[c] += M[c][d] * v[d];
        }
        uint64_t mx = 0;
        for (int c = 0; c < nc; ++c) {
            uint64_t a = (uint64_t)(w[c] < 0 ? -w[c] : w[c]);
            if (a > mx) mx = a;
        }
        if (mx == 0) {
            if (it == 0) for (int c = 0; c < nc; ++c) v[c] = 1;
            break;
        }
        const int s = bitlen64(mx) > 20 ? bitlen64(mx) - 20 : 0;
        for (int c = 0; c < nc; ++c) {
            const uint64_t a = (uint64_t)(w[c] < 0 ? -w[c] : w[c]) >> s;
            v[c] = w[c] < 0 ? -(int64_t)a : (int64_t)a;
        }
    }
    int first = 1;
    int64_t dmin = 0, dmax = 0;
    *imin = *imax = 0;
    for (int i = 0; i < 16; ++i) {
        if (!((mask >> i) & 1u)) continue;
        int64_t d = 0;
        for (int c = 0; c < nc; ++c) d += (int64_t)px[4 * i + chs[c]] * v[c];
        if (first || d < dmin) { dmin = d; *imin = i; }
        if (first || d > dmax) { dmax = d; *imax = i; }
        first = 0;
    }
}

/* nearest code of `bits` bits (plus p-bit p >= 0) to the 8-bit value e */
static int nearest_code(int e, int bits, int p)
{
    int best = -1, bk = 0;
    for (int k = 0; k < (1 << bits); ++k) {
        int val = p < 0 ? expand8(k, bits) : expand8((k << 1) | p, bits + 1);
        int d = val > e ? val - e : e - val;
        if (best < 0 || d < best) { best = d; bk = k; }
    }
    return bk;
}

static int64_t block_sse(const uint8_t blk[16], const uint8_t px[64])
{
    uint8_t dec[64];
    oracle_bc7_decode_block(blk, dec);
    int64_t e = 0;
    for (int i = 0; i < 64; ++i) e += (int64_t)(dec[i] - px[i]) * (dec[i] - px[i]);
    return e;
}

static void encode_mode5(const uint8_t in[64], int rot, uint8_t out[16])
{
    uint8_t px[64];
    memcpy(px, in, 64);
    if (rot > 0)
        for (int i = 0; i < 16; ++i) { uint8_t t = px[4 * i + 3]; px[4 * i + 3] = px[4 * i + rot - 1]; px[4 * i + rot - 1] = t; }
    const int rgb[3] = {0, 1, 2};
    int imin, imax;
    axis_extremes(px, 0xffffu, rgb, 3, &imin, &imax);
    int C0[3], C1[3], V0[3], V1[3];
    for (int c = 0; c < 3; ++c) {
        C0[c] = nearest_code(px[4 * imin + c], 7, -1);
        C1[c] = nearest_code(px[4 * imax + c], 7, -1);
        V0[c] = expand8(C0[c], 7);
        V1[c] = expand8(C1[c], 7);
    }
    int A0 = 255, A1 = 0;
    for (int i = 0; i < 16; ++i) {
        if (px[4 * i + 3] < A0) A0 = px[4 * i + 3];
        if (px[4 * i + 3] > A1) A1 = px[4 * i + 3];
    }
    int ci[16], ai[16];
    for (int i = 0; i < 16; ++i) {
        int best = -1, ba = -1;
        for (int w = 0; w < 4; ++w) {
            int err = 0;
            for (int c = 0; c < 3; ++c) {
                const int d = interp(V0[c], V1[c], BC7_W2[w]) - px[4 * i + c];
                err += d * d;
            }
            if (best < 0 || err < best) { best = err; ci[i] = w; }
            const int da = interp(A0, A1, BC7_W2[w]) - px[4 * i + 3];
            if (ba < 0 || da * da < ba) { ba = da * da; ai[i] = w; }
        }
    }
    if (ci[0] >= 2) {
        for (int c = 0; c < 3; ++c) { int t = C0[c]; C0[c] = C1[c]; C1[c] = t; }
        for (int i = 0; i < 16; ++i) ci[i] = 3 - ci[i];
    }
    if (ai[0] >= 2) {
        int t = A0; A0 = A1; A1 = t;
        for (int i = 0; i < 16; ++i) ai[i] = 3 - ai[i];
    }
    memset(out, 0, 16);
    bitwriter bw = {out, 0};
    put(&bw, 1 << 5, 6);
    put(&bw, rot, 2);
    for (int c = 0; c < 3; ++c) { put(&bw, C0[c], 7); put(&bw, C1[c], 7); }
    put(&bw, A0, 8);
    put(&bw, A1, 8);
    put(&bw, ci[0], 1);
    for (int i = 1; i < 16; ++i) put(&bw, ci[i], 2);
    put(&bw, ai[0], 1);
    for (int i = 1; i < 16; ++i) put(&bw, ai[i], 2);
}

static void encode_mode7(const uint8_t px[64], int part, uint8_t out[16])
{
    const int rgba[4] = {0, 1, 2, 3};
    int code[2][2][4], pb[2][2], val[2][2][4], idx[16];
    uint32_t mask[2] = {0, 0};
    for (int i = 0; i < 16; ++i) mask[oracle_bc7_subset(2, part, i)] |= 1u << i;
    for (int s = 0; s < 2; ++s) {
        int ie[2];
        axis_extremes(px, mask[s], rgba, 4, &ie[0], &ie[1]);
        for (int e = 0; e < 2; ++e) {
            int best = -1;
            for (int p = 0; p < 2; ++p) {
                int k[4], err = 0;
                for (int c = 0; c < 4; ++c) {
                    k[c] = nearest_code(px[4 * ie[e] + c], 5, p);
                    const int d = expand8((k[c] << 1) | p, 6) - px[4 * ie[e] + c];
                    err += d * d;
                }
                if (best < 0 || err < best) {
                    best = err;
                    pb[s][e] = p;
                    for (int c = 0; c < 4; ++c) { code[s][e][c] = k[c]; val[s][e][c] = expand8((k[c] << 1) | p, 6); }
                }
            }
        }
    }
    for (int i = 0; i < 16; ++i) {
        const int s = oracle_bc7_subset(2, part, i);
        int best = -1;
        for (int w = 0; w < 4; ++w) {
            int err = 0;
            for (int c = 0; c < 4; ++c) {
                const int d = interp(val[s][0][c], val[s][1][c], BC7_W2[w]) - px[4 * i + c];
                err += d * d;
            }
            if (best < 0 || err < best) { best = err; idx[i] = w; }
        }
    }
    for (int s = 0; s < 2; ++s) {
        const int a = oracle_bc7_anchor(2, part, s);
        if (idx[a] >= 2) {
            for (int c = 0; c < 4; ++c) { int t = code[s][0][c]; code[s][0][c] = code[s][1][c]; code[s][1][c] = t; }
            int t = pb[s][0]; pb[s][0] = pb[s][1]; pb[s][1] = t;
            for (int i = 0; i < 16; ++i)
                if (oracle_bc7_subset(2, part, i) == s) idx[i] = 3 - idx[i];
        }
    }
    memset(out, 0, 16);
    bitwriter bw = {out, 0};
    put(&bw, 1 << 7, 8);
    put(&bw, part, 6);
    for (int c = 0; c < 4; ++c)
        for (int s = 0; s < 2; ++s)
            for (int e = 0; e < 2; ++e) put(&bw, code[s][e][c], 5);
    for (int s = 0; s < 2; ++s)
        for (int e = 0; e < 2; ++e) put(&bw, pb[s][e], 1);
    const int a1 = oracle_bc7_anchor(2, part, 1);
    for (int i = 0; i < 16; ++i) put(&bw, idx[i], (i == 0 || i == a1) ? 1 : 2);
}

/* returns the chosen mode (6, 5 or 7) */
int oracle_bc7_encode_multi(const uint8_t px[64], uint8_t out[16])
{
    uint8_t cand[16];
    oracle_bc7_encode_mode6(px, out);
    int64_t best = block_sse(out, px);
    int mode = 6;
    for (int r = 0; r < 4 && best > 0; ++r) {
        encode_mode5(px, r, cand);
        const int64_t e = block_sse(cand, px);
        if (e < best) { best = e; memcpy(out, cand, 16); mode = 5; }
    }
    for (int p = 0; p < 64 && best > 0; ++p) {
        encode_mode7(px, p, cand);
        const int64_t e = block_sse(cand, px);
        if (e < best) { best = e; memcpy(out, cand, 16); mode = 7; }
    }
    return mode;
}

void oracle_bc7_encode_image_multi(const uint8_t *rgba, int w, int h, uint8_t *blocks)
{
    for (int by = 0; by < h / 4; ++by)
        for (int bx = 0; bx < w / 4; ++bx) {
            uint8_t px[64];
            for (int i = 0; i < 16; ++i)
                memcpy(px + 4 * i, rgba + ((size_t)(4 * by + i / 4) * w + 4 * bx + i % 4) * 4, 4);
            oracle_bc7_encode_multi(px, blocks + ((size_t)by * (w / 4) + bx) * 16);
        }
}
