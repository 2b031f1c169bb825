// kern_nest.cu -- general affine loop-nest kernels, one per operator pair.
#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstring>

#include "lsb_dispatch.cuh"
#include "nest_fast.cuh"

namespace lsb {

// ---- fast path (nest_fast.cuh) ---------------------------------------------
namespace {
// |base| + sum |coeff| (extent - 1) of an affine form over the padded dims, or -1 past 31 bits
bool pack_affine(const lsb_nest_desc &d, const lsb_affine &f, NfAffine *out) {
    const int so = kNfOut - d.n_out, sr = kNfRed - d.n_red;
    int64_t span = f.base < 0 ? -f.base : f.base;
    memset(out, 0, sizeof(*out));
    for (int i = 0; i < d.n_out + d.n_red; i++) {
        const int64_t c = f.coeff[i];
        span += (c < 0 ? -c : c) * (d.extent[i] - 1);
        if (c > INT32_MAX || c < INT32_MIN) return false;
        if (i < d.n_out) out->co[so + i] = (int)c;
        else out->cr[sr + i - d.n_out] = (int)c;
    }
    if (span >= INT32_MAX || f.base > INT32_MAX || f.base < INT32_MIN) return false;
    out->base = (int)f.base;
    return true;
}

template <int NOPS, bool GUARDS, bool RED>
void launch_rows(const NestFastArgs &a, dim3 grid, int tx_log2, cudaStream_t s) {
    nest_rows_kernel<NOPS, GUARDS, RED><<<grid, 256, 0, s>>>(a, tx_log2);
}
}  // namespace

int launch_nest_fast(const lsb_nest_desc &d, const EpiStages &epi, cudaStream_t s) {
    if (d.n_out > kNfOut || d.n_red > kNfRed || d.n_operands > kNfOps) return 0;
    NestFastArgs a;
    memset(&a, 0, sizeof(a));
    const int so = kNfOut - d.n_out, sr = kNfRed - d.n_red;
    int64_t points = 1, red = 1;
    for (int i = 0; i < kNfOut; i++) a.eo[i] = 1;
    for (int i = 0; i < kNfRed; i++) a.er[i] = 1;
    for (int i = 0; i < d.n_out + d.n_red; i++) {
        if (d.extent[i] >= INT32_MAX) return 0;
        if (i < d.n_out) { a.eo[so + i] = (int)d.extent[i]; points *= d.extent[i]; }
        else { a.er[sr + i - d.n_out] = (int)d.extent[i]; red *= d.extent[i]; }
    }
    if (points >= INT32_MAX || red >= INT32_MAX) return 0;
    a.shift = so;
    a.n_rows = a.eo[0] * a.eo[1] * a.eo[2];
    bool guards = false;
    for (int o = 0; o < d.n_operands; o++) {
        const lsb_nest_operand &src = d.operand[o];
        if (src.n_guards > kNfGuards) return 0;
        a.op[o].ptr = src.ptr;
        a.op[o].fill = src.fill;
        a.op[o].n_guards = src.n_guards;
        if (!pack_affine(d, src.addr, &a.op[o].addr)) return 0;
        for (int q = 0; q < src.n_guards; q++) {
            if (!pack_affine(d, src.guard[q], &a.op[o].guard[q])) return 0;
            if (src.guard_size[q] < 0 || src.guard_size[q] > INT32_MAX) return 0;
            a.op[o].guard_size[q] = (unsigned)src.guard_size[q];
            guards = true;
        }
    }
    if (!pack_affine(d, d.out_addr, &a.out_addr)) return 0;
    a.out = d.out;
    a.beta = d.beta;
    a.combine = d.combine;
    a.reduce = d.reduce;
    a.epi = epi;
    const int inner = a.eo[3];
    // permutation of a single operand: 32 x 64 smem tiles
    if (d.n_red == 0 && d.n_operands == 1 && !guards && epi.n == 0 && d.beta == 1.0f && a.out_addr.co[3] == 1 &&
        a.op[0].addr.co[3] != 1 && inner >= 16) {
        int q = -1;
        for (int i = 0; i < 3; i++)
            if (a.op[0].addr.co[i] == 1 && a.eo[i] >= 16) q = i;
        if (q >= 0) {
            a.tq = q;
            a.tb0 = q == 0 ? 1 : 0;
            a.tb1 = q == 2 ? 1 : 2;
            const int64_t batch = (int64_t)a.eo[a.tb0] * a.eo[a.tb1];
            // both sides in whole float4s: 64 x 64 tiles
            const NfAffine &fi = a.op[0].addr, &fo = a.out_addr;
            const bool v4 = inner % 4 == 0 && a.eo[q] % 4 == 0 && fi.base % 4 == 0 && fi.co[3] % 4 == 0 &&
                            fi.co[a.tb0] % 4 == 0 && fi.co[a.tb1] % 4 == 0 && fo.base % 4 == 0 && fo.co[q] % 4 == 0 &&
                            fo.co[a.tb0] % 4 == 0 && fo.co[a.tb1] % 4 == 0 && ((uintptr_t)a.out & 15) == 0 &&
                            ((uintptr_t)a.op[0].ptr & 15) == 0;
            if (v4 && (a.eo[q] + 63) / 64 <= 65535) {
                dim3 g4((unsigned)((inner + 63) / 64), (unsigned)((a.eo[q] + 63) / 64),
                        (unsigned)std::min<int64_t>(batch, 65535));
                nest_transpose4_kernel<<<g4, 256, 0, s>>>(a);
                return 5;
            }
            dim3 grid((unsigned)((inner + kNfTileI - 1) / kNfTileI), (unsigned)((a.eo[q] + kNfTileQ - 1) / kNfTileQ),
                      (unsigned)std::min<int64_t>(batch, 65535));
            if (grid.y <= 65535) {
                nest_transpose_kernel<<<grid, 256, 0, s>>>(a);
                return 2;
            }
        }
    }
    // elementwise / broadcast / concat rows, 16-byte aligned: float4 groups
    if (d.n_red == 0 && epi.n == 0 && a.out_addr.co[3] == 1 && inner % 4 == 0) {
        auto quad = [](const NfAffine &f) { return f.base % 4 == 0 && f.co[0] % 4 == 0 && f.co[1] % 4 == 0 && f.co[2] % 4 == 0; };
        bool ok = quad(a.out_addr) && ((uintptr_t)a.out & 15) == 0;
        for (int o = 0; o < d.n_operands; o++) {
            const int c3 = a.op[o].addr.co[3];
            ok = ok && (c3 == 0 || (c3 == 1 && quad(a.op[o].addr) && ((uintptr_t)a.op[o].ptr & 15) == 0));
        }
        if (ok) {
            const int inner4 = inner / 4;
            int lg = 3;
            while (lg < 8 && (1 << lg) < inner4) lg++;
            const int TX = 1 << lg, TY = 256 >> lg;
            const int64_t row_blocks = ((int64_t)a.n_rows + TY - 1) / TY;
            int64_t gx = ((int64_t)inner4 + 4 * TX - 1) / (4 * TX);
            if (gx * row_blocks < 4 * (int64_t)device_sms()) gx = ((int64_t)inner4 + TX - 1) / TX;
            dim3 grid((unsigned)gx, (unsigned)std::min<int64_t>(row_blocks, 65535));
            if (d.n_operands == 1) {
                if (guards) nest_vec4_guarded_kernel<1><<<grid, 256, 0, s>>>(a, lg);
                else nest_vec4_kernel<1><<<grid, 256, 0, s>>>(a, lg);
            } else {
                if (guards) nest_vec4_guarded_kernel<2><<<grid, 256, 0, s>>>(a, lg);
                else nest_vec4_kernel<2><<<grid, 256, 0, s>>>(a, lg);
            }
            return 3;
        }
    }
    // non-overlapping pooling along the innermost dim, 16-byte aligned rows
    if (d.n_red > 0 && d.n_operands == 1 && !guards && epi.n == 0 && a.out_addr.co[3] == 1 && inner % 4 == 0 &&
        a.op[0].addr.cr[2] == 1 && a.er[2] == a.op[0].addr.co[3] && (a.er[2] == 2 || a.er[2] == 4)) {
        auto quad = [](const NfAffine &f) {
            return f.base % 4 == 0 && f.co[0] % 4 == 0 && f.co[1] % 4 == 0 && f.co[2] % 4 == 0 && f.cr[0] % 4 == 0 &&
                   f.cr[1] % 4 == 0;
        };
        if (quad(a.out_addr) && quad(a.op[0].addr) && ((uintptr_t)a.out & 15) == 0 && ((uintptr_t)a.op[0].ptr & 15) == 0) {
            const int inner4 = inner / 4;
            int lg = 3;
            while (lg < 8 && (1 << lg) < inner4) lg++;
            const int TX = 1 << lg, TY = 256 >> lg;
            const int64_t row_blocks = ((int64_t)a.n_rows + TY - 1) / TY;
            int64_t gx = ((int64_t)inner4 + 4 * TX - 1) / (4 * TX);
            if (gx * row_blocks < 4 * (int64_t)device_sms()) gx = ((int64_t)inner4 + TX - 1) / TX;
            dim3 grid((unsigned)gx, (unsigned)std::min<int64_t>(row_blocks, 65535));
            if (a.er[2] == 2) nest_pool_kernel<2><<<grid, 256, 0, s>>>(a, lg);
            else nest_pool_kernel<4><<<grid, 256, 0, s>>>(a, lg);
            return 4;
        }
    }
    int tx_log2 = 3;
    while (tx_log2 < 8 && (1 << tx_log2) < inner) tx_log2++;
    const int TX = 1 << tx_log2, TY = 256 >> tx_log2;
    const int64_t row_blocks = ((int64_t)a.n_rows + TY - 1) / TY;
    const bool red_loop = d.n_red > 0;
    const int per_trip = red_loop ? 4 : 8;
    int64_t gx = ((int64_t)inner + per_trip * TX - 1) / (per_trip * TX);
    if (gx * row_blocks < 4 * (int64_t)device_sms()) gx = ((int64_t)inner + TX - 1) / TX;
    dim3 grid((unsigned)gx, (unsigned)std::min<int64_t>(row_blocks, 65535));
    const int key = (d.n_operands == 2 ? 4 : 0) | (guards ? 2 : 0) | (red_loop ? 1 : 0);
    switch (key) {
    case 0: launch_rows<1, false, false>(a, grid, tx_log2, s); break;
    case 1: launch_rows<1, false, true>(a, grid, tx_log2, s); break;
    case 2: launch_rows<1, true, false>(a, grid, tx_log2, s); break;
    case 3: launch_rows<1, true, true>(a, grid, tx_log2, s); break;
    case 4: launch_rows<2, false, false>(a, grid, tx_log2, s); break;
    case 5: launch_rows<2, false, true>(a, grid, tx_log2, s); break;
    case 6: launch_rows<2, true, false>(a, grid, tx_log2, s); break;
    default: launch_rows<2, true, true>(a, grid, tx_log2, s); break;
    }
    return 1;
}

template <int C, int R>
void launch_nest(const NestArgs &a, cudaStream_t s) {
    int64_t blocks = std::min<int64_t>((a.n_points + 255) / 256, (int64_t)device_sms() * 16);
    affine_nest_kernel<C, R><<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, s>>>(a);
}

#define NEST_ROW(C) {launch_nest<C, 0>, launch_nest<C, 1>, launch_nest<C, 2>, launch_nest<C, 3>}
const NestFn kNest[4][4] = {NEST_ROW(0), NEST_ROW(1), NEST_ROW(2), NEST_ROW(3)};
#undef NEST_ROW

}  // namespace lsb
