// slab.hpp — x-slab decomposition of a 2D / 3D dealiased convolution over G ranks.
//
// Backend-agnostic: the driver below owns the index arithmetic and the schedule; the library
// that instantiates it supplies the local compute, memory, copies and the exchange (`Ops`).
//   libhconv_cuda.so   Ops = device buffers, sm_100a kernels, NCCL (or a callback) on a
//                      plan-owned communication stream, events between the two streams
//   libhconv_oracle.so Ops = host buffers, the oracle's padded FFTs, the callback (gloo in the
//                      CPU tests), synchronous -- the same index arithmetic, checked on CPU
//
// The reference has no distributed code; the decomposition extends convolve_nd
// (PAPER.md:584-600).  Global arrays [x][y] or [x][y][z] (z innermost, the
// Hermitian axis in Hermitian mode, x and y centered) are split into x-slabs;
// rank g owns rows [x0_g, x0_g + nx_g).  A padded FFT needs its whole axis, so the OUTER padded
// transform runs along y, which every rank holds completely, and x becomes an inner axis after
// one transpose.  For each residue r of the y axis:
//   1. forward padded y-FFT of the A input slabs, written k-major F_a[k][x][z] (k < B_y): the
//      k-rows destined for rank h are one contiguous run (no packing before the exchange);
//   2. all-to-all in chunks of k-rows: rank g receives, from every h, the rows k of its own
//      k-range K_g for h's x-rows, R_a[c][h][k][x_h][z]; one strided copy per (chunk, peer)
//      places them as T_a[k][x][z] with x complete;
//   3. the (d-1)-D subconvolutions of the chunk's k-lines (x, or x then z) in one batched call,
//      outputs in T_b (b < B);
//   4. strided copies back into the send layout and the all-to-all back: W_b[k][x_g][z];
//   5. inverse padded y-FFT of residue r accumulated into the output slab (last residue scaled
//      by 1/(q_y m_y)).
// The multi-D DFT is separable and the inner subconvolutions are pointwise in the y frequency,
// so this is the paper's recursion with the roles of x and y exchanged.  Chunk c's exchange
// overlaps chunk c-1's subconvolutions and chunk c-2's exchange back (CUDA: two streams).
#pragma once
#include <algorithm>
#include <cstddef>
#include <stdexcept>
#include <vector>

#include "../../include/hconv.h"

namespace hslab {

struct Range {
  size_t lo = 0, hi = 0;
  size_t size() const { return hi - lo; }
};

// Balanced contiguous split of [0, n) into `parts` ranges (uneven: 511 = 7*64 + 63).
inline std::vector<Range> partition(size_t n, size_t parts) {
  std::vector<Range> out(parts);
  const size_t base = n / parts, extra = n % parts;
  size_t lo = 0;
  for (size_t g = 0; g < parts; ++g) {
    const size_t hi = lo + base + (g < extra ? 1 : 0);
    out[g] = {lo, hi};
    lo = hi;
  }
  return out;
}

// Geometry shared by every rank (each rank computes the same values from the descriptor).
struct Geometry {
  int G = 1, rank = 0;
  size_t Lx = 0, Ly = 0, Z = 1;  // stored extents of x, y and the innermost axis (1 in 2D)
  size_t By = 0;                 // y block length (natural order), the spectral rows per residue
  size_t ny_res = 1;             // residues of the y axis
  double scale = 1.0;            // 1 / (q_y m_y)
  size_t nchunks = 1;            // k-chunks per exchange (the same on every rank)
  std::vector<Range> xs, ks;     // x-slab and k-range of every rank
  size_t nx() const { return xs[rank].size(); }
  size_t nk() const { return ks[rank].size(); }
  // chunk c of rank h's k-range, relative to ks[h].lo
  Range chunk(int h, size_t c) const { return partition(ks[h].size(), nchunks)[c]; }
  size_t max_chunk() const {
    size_t m = 0;
    for (size_t c = 0; c < nchunks; ++c) m = std::max(m, chunk(rank, c).size());
    return m;
  }
};

inline Geometry make_geometry(int rank, int G, size_t Lx, size_t Ly, size_t Z, size_t By, size_t ny_res,
                              double scale, size_t chunks_req) {
  if (G < 1 || rank < 0 || rank >= G) throw std::invalid_argument("slab: bad rank / rank count");
  Geometry g;
  g.G = G;
  g.rank = rank;
  g.Lx = Lx;
  g.Ly = Ly;
  g.Z = Z;
  g.By = By;
  g.ny_res = ny_res;
  g.scale = scale;
  g.xs = partition(Lx, (size_t)G);
  g.ks = partition(By, (size_t)G);
  // default: 4 chunks (enough to overlap the exchanges with the subconvolutions, few enough that
  // every message stays large); never more chunks than the smallest rank has k-rows
  size_t nc = chunks_req ? chunks_req : 4;
  size_t kmin = By;
  for (const Range& r : g.ks) kmin = std::min(kmin, r.size());
  g.nchunks = std::max<size_t>(1, std::min(nc, std::max<size_t>(1, kmin)));
  return g;
}

// Ops contract (see the file comment):
//   void* alloc(size_t elems)                 complex128 elements; free(void*)
//   void fwd(size_t r, const void* f, void* F)  forward y residue r of the x-slab into F[k][x][z]
//   void bwd(size_t r, const void* W, void* h, bool acc, double scale)   inverse into the slab
//   void inner(size_t count, void* const* T)  (d-1)-D subconvolutions of `count` contiguous
//                                             [x][z] arrays, in place (outputs over the first B)
//   void copy2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
//               size_t rows, bool on_comm)   pitches / width in elements
//   void exchange(const void* send, const size_t* sc, const size_t* sd, void* recv,
//                 const size_t* rc, const size_t* rd)   on the communication side
//   void comm_after_compute(), compute_after_comm(size_t tag), mark_comm(size_t tag)
//                                             stream ordering (no-ops when synchronous)
template <class Ops>
class Driver {
 public:
  Driver(const Geometry& g, size_t A, size_t B, Ops& ops) : g_(g), A_(A), B_(B), ops_(ops) {
    const size_t nxz = g.nx() * g.Z, spec = g.By * nxz;
    const size_t tk = g.max_chunk() * g.Lx * g.Z;
    for (size_t a = 0; a < A; ++a) {
      F_.push_back(ops.alloc(std::max<size_t>(1, spec)));
      R_.push_back(ops.alloc(std::max<size_t>(1, g.nk() * g.Lx * g.Z)));
    }
    // T: one chunk of complete x-lines per operand (max(A, B)); S: the send-back layout
    for (size_t i = 0; i < std::max(A, B); ++i) T_.push_back(ops.alloc(std::max<size_t>(1, tk)));
    for (size_t b = 0; b < B; ++b) {
      S_.push_back(ops.alloc(std::max<size_t>(1, g.nk() * g.Lx * g.Z)));
      W_.push_back(ops.alloc(std::max<size_t>(1, spec)));
    }
  }
  ~Driver() {
    for (auto* v : {&F_, &R_, &T_, &S_, &W_})
      for (void* p : *v) ops_.free(p);
  }
  Driver(const Driver&) = delete;
  Driver& operator=(const Driver&) = delete;

  size_t buffer_elems() const {
    const size_t nxz = g_.nx() * g_.Z, spec = g_.By * nxz, rk = g_.nk() * g_.Lx * g_.Z;
    return A_ * (spec + rk) + std::max(A_, B_) * g_.max_chunk() * g_.Lx * g_.Z + B_ * (rk + spec);
  }

  // in[A], acc[B]: this rank's slabs; acc must not alias an input (the caller copies back)
  void run(const void* const* in, void* const* acc) {
    const Geometry& g = g_;
    const size_t G = (size_t)g.G, Z = g.Z, nx = g.nx(), nxz = nx * Z;
    // per (chunk, peer) counts and displacements of both exchanges, in elements
    std::vector<size_t> sc(G), sd(G), rc(G), rd(G), bc(G), bd(G), wc(G), wd(G);
    for (size_t r = 0; r < g.ny_res; ++r) {
      for (size_t a = 0; a < A_; ++a) ops_.fwd(r, in[a], F_[a]);
      ops_.comm_after_compute();
      // forward exchanges of every chunk, in order, on the communication side
      for (size_t c = 0; c < g.nchunks; ++c) {
        const size_t roff = chunk_roff(c);
        for (size_t h = 0; h < G; ++h) {
          const Range kc = g.chunk((int)h, c);  // rows of rank h's k-range I send to h
          sc[h] = kc.size() * nxz;
          sd[h] = (g.ks[h].lo + kc.lo) * nxz;
          const Range mine = g.chunk(g.rank, c);
          rc[h] = mine.size() * g.xs[h].size() * Z;
          rd[h] = roff + mine.size() * g.xs[h].lo * Z;
        }
        for (size_t a = 0; a < A_; ++a) ops_.exchange(F_[a], sc.data(), sd.data(), R_[a], rc.data(), rd.data());
        ops_.mark_comm(c);
      }
      // per chunk: place, subconvolve, unplace, exchange back
      for (size_t c = 0; c < g.nchunks; ++c) {
        const Range mine = g.chunk(g.rank, c);
        const size_t cnt = mine.size(), roff = chunk_roff(c);
        ops_.compute_after_comm(c);
        if (cnt) {
          for (size_t a = 0; a < A_; ++a)
            for (size_t h = 0; h < G; ++h) {
              const size_t w = g.xs[h].size() * Z;
              if (w)
                ops_.copy2d((char*)T_[a] + 16 * g.xs[h].lo * Z, g.Lx * Z,
                            (const char*)R_[a] + 16 * (roff + cnt * g.xs[h].lo * Z), w, w, cnt, false);
            }
          ops_.inner(cnt, T_.data());
          for (size_t b = 0; b < B_; ++b)
            for (size_t h = 0; h < G; ++h) {
              const size_t w = g.xs[h].size() * Z;
              if (w)
                ops_.copy2d((char*)S_[b] + 16 * (roff + cnt * g.xs[h].lo * Z), w,
                            (const char*)T_[b] + 16 * g.xs[h].lo * Z, g.Lx * Z, w, cnt, false);
            }
        }
        ops_.comm_after_compute();
        for (size_t h = 0; h < G; ++h) {
          bc[h] = cnt * g.xs[h].size() * Z;  // what I computed for h's x-rows
          bd[h] = roff + cnt * g.xs[h].lo * Z;
          const Range kc = g.chunk((int)h, c);  // h's chunk of its k-range, my x-rows
          wc[h] = kc.size() * nxz;
          wd[h] = (g.ks[h].lo + kc.lo) * nxz;
        }
        for (size_t b = 0; b < B_; ++b) ops_.exchange(S_[b], bc.data(), bd.data(), W_[b], wc.data(), wd.data());
      }
      ops_.compute_after_comm((size_t)-1);
      const bool last = r + 1 == g.ny_res;
      for (size_t b = 0; b < B_; ++b) ops_.bwd(r, W_[b], acc[b], r > 0, last ? g.scale : 1.0);
    }
  }

 private:
  // element offset of chunk c in R / S (chunk-major: [c][h][k][x_h][z])
  size_t chunk_roff(size_t c) const { return g_.chunk(g_.rank, c).lo * g_.Lx * g_.Z; }

  Geometry g_;
  size_t A_, B_;
  Ops& ops_;
  std::vector<void*> F_, R_, T_, S_, W_;
};

}  // namespace hslab
