// store callback for tools/cufft_cb_pack_probe.cu: the 2-D D2Z output element
// (c, xl, ky, kz) goes straight to the x-pencil layout of its destination
// slab j = ky / nyl (what k_pack / k_pack_peer do after the transform).
#include <cufftXt.h>

struct PackCb {
    double2* const* peer;  // destination spectrum of every slab
    unsigned nzh, ny, nxl, nyl;
    unsigned long long blk;  // elements per source-slab block in a destination (nxl * 6 * nyl * nzh)
    unsigned rank;
};

__device__ void cb_pack_store(void* out, unsigned long long off, cufftDoubleComplex v, void* info, void* sh) {
    const PackCb* p = static_cast<const PackCb*>(info);
    const unsigned o = (unsigned)off;
    const unsigned kz = o % p->nzh, t = o / p->nzh;
    const unsigned ky = t % p->ny, cx = t / p->ny;
    const unsigned c = cx / p->nxl, xl = cx - c * p->nxl;
    const unsigned j = ky / p->nyl, kyl = ky - j * p->nyl;
    p->peer[j][p->rank * p->blk + ((unsigned long long)(xl * 6 + c) * p->nyl + kyl) * p->nzh + kz] = v;
}
