// Tile spaces of the persistent scan: slot -> tile decoding, shared by the
// kernels (scan_kernels.cu) and the host-side planner the multi-rank tests use
// (tsd_tile_plan), so both deal the same tiles to the same ranks.
#pragma once

#include "common.cuh"

namespace tsd {

__host__ __device__ __forceinline__ int tile_imin(int a, int b) { return a < b ? a : b; }

// Launch-invariant tile-space values, read from the control block once per
// CTA (the previous kernels of the try wrote them): the tile loop then decodes
// a slot with one load (its group) instead of a chain of control-block loads.
struct TileCtx {
    long long slots;  // tile slots of the launch
    long long G;      // groups (band / tracked / full spaces)
    long long nf;     // catch-all: far bands [tK0, N) still to run
    long long k0;     // band / tracked spaces: first diagonal of band 0
};

// Slot -> tile.  Band spaces are band-major (near bands first), full rows are
// distance-major across groups (near tiles of every group first), so kills
// from near diagonals land before the far tiles are fetched.
__host__ __device__ __forceinline__ bool tile_decode(const ScanParams& p, const TileCtx& c, long long t, TileDesc& td) {
    const int N = p.N;
    const int side = (int)(t & 1);
    int a, e;
    long long k0;
    if (p.space == kSpaceSeed) {
        if (p.nb == 1) t <<= 1;  // one-sided band 0: positive side only
        const int j = (int)(t >> 1);
        a = j * p.L;
        e = tile_imin(N, a + p.L) - 1;
        td.r0 = a;
        td.rows = e - a + 1;
        if (side == 0) {
            if ((long long)a + p.kA >= N) return false;
            td.k0 = p.kA;
            td.dir = +1;
            td.seed = 2 * j;
        } else {
            if ((long long)e - p.kA < 0) return false;
            td.k0 = -p.kA - kW + 1;
            td.dir = -1;
            td.seed = td.rows == p.L ? 2 * j + 1 : -1;
        }
        return true;
    }
    td.seed = -1;
    const long long G = c.G;
    long long b, gi;  // band and group of the slot (32-bit division when it fits: no 64-bit emulation)
    if (c.slots <= 0xffffffffll) {
        const unsigned tt = (unsigned)t, g1 = (unsigned)G;
        b = tt / (2u * g1);
        gi = (tt >> 1) % g1;
    } else {
        b = t / (2 * G);
        gi = (t >> 1) % G;
    }
    if (p.space == kSpaceBlocks) {
        const int g = (int)gi;
        a = g * p.L;
        e = tile_imin(N, a + p.L) - 1;
        k0 = c.k0 + b * kW;
    } else if (p.space == kSpaceBand || p.space == kSpaceTrack || p.space == kSpaceTrackRest) {
        const int2 gr = p.groups[gi];
        a = gr.x;
        e = gr.y;
        if (p.space == kSpaceTrackRest) k0 = b < c.nf ? c.k0 + b * kW : (long long)p.m + (b - c.nf) * kW;
        else k0 = c.k0 + b * kW;
    } else {
        const int2 gr = p.groups[gi];
        a = gr.x;
        e = gr.y;
        td.r0 = a;
        td.rows = e - a + 1;
        if (side == 0) {  // k in [m, N-1-a]
            if ((long long)p.m + b * kW > (long long)N - 1 - a) return false;
            td.k0 = p.m + (int)b * kW;
            td.dir = +1;
        } else {  // k in [-e, -m]
            const long long khi = -(long long)p.m - b * kW;
            if (e + khi < 0) return false;
            td.k0 = (int)(khi - kW + 1);
            td.dir = -1;
        }
        return true;
    }
    td.r0 = a;
    td.rows = e - a + 1;
    if (side == 0) {
        if (a + k0 >= N) return false;
        td.k0 = (int)k0;
        td.dir = +1;
    } else {
        if (e - k0 < 0) return false;
        td.k0 = (int)(-k0 - kW + 1);
        td.dir = -1;
    }
    return true;
}

}  // namespace tsd
