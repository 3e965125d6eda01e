// Marching cubes over the device volume (the reference's
// refusion/meshing.py:112-245, `marching_cubes`).
//
// One CTA per block, one thread per cell (cell l = x + 8y + 64z, anchored at
// voxel l; its +x/+y/+z corners spill into up to seven neighbour blocks,
// meshing.py:112-146).  Blocks are visited in sorted key order (= sorted
// coordinate order, meshing.py:229-231) and cells in l order, so a count
// pass, an exclusive scan over blocks and an emit pass reproduce the
// reference's vertex and triangle order exactly.  Per cell (meshing.py:
// 149-213): all eight corners observed (W > 0), case bit i = D_i < 0, one
// vertex per cut edge in edge order, t = da / (da - db) (0.5 when equal),
// position pa + t (pb - pa), colour ca + t (cb - ca), triangles indexing the
// cell's vertices by the cut edge's rank.  IEEE f64, no contraction.
#pragma once

#include "rf_kernels.cuh"

#include <math_constants.h>

namespace rf {

// Corner i of a cell: (x, y, z) offsets (meshing.py:23-35)
__constant__ int kMcCorner[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                                    {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};
// Edge e joins corners (a, b) (mc_tables.py:10-23)
__constant__ int kMcEdge[12][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 0}, {4, 5}, {5, 6},
                                   {6, 7}, {7, 4}, {0, 4}, {1, 5}, {2, 6}, {3, 7}};
// Triangle lists of the 256 cases, packed by tools/gen_mc_table.py from the
// canonical table (mc_tables.py:44-302): nibble i = i-th edge, bits 60-63 =
// triangle count.
__constant__ unsigned long long kMcTriangles[256] = {
    0x0000000000000000ull, 0x1000000000000380ull, 0x1000000000000910ull, 0x2000000000189381ull,
    0x1000000000000a21ull, 0x2000000000a21380ull, 0x2000000000920a29ull, 0x300000089a8a2382ull,
    0x10000000000002b3ull, 0x20000000000b82b0ull, 0x2000000000b32091ull, 0x3000000b89b912b1ull,
    0x20000000003ab1a3ull, 0x3000000ab8a801a0ull, 0x30000009ab9b3093ull, 0x2000000000b8aa89ull,
    0x1000000000000874ull, 0x2000000000437034ull, 0x2000000000748910ull, 0x3000000137174914ull,
    0x2000000000748a21ull, 0x3000000a21403743ull, 0x3000000748209a29ull, 0x40004973727929a2ull,
    0x20000000002b3748ull, 0x300000040242b74bull, 0x3000000b32748109ull, 0x40001292b9b49b74ull,
    0x3000000487ab31a3ull, 0x40004b7401b41ab1ull, 0x400030bab9b09874ull, 0x3000000ab99b4b74ull,
    0x1000000000000459ull, 0x2000000000380459ull, 0x2000000000051450ull, 0x3000000513538458ull,
    0x2000000000459a21ull, 0x3000000594a21803ull, 0x3000000204245a25ull, 0x40008434535235a2ull,
    0x2000000000b32459ull, 0x3000000594b802b0ull, 0x3000000b32510450ull, 0x4000584b82852512ull,
    0x300000045931ab3aull, 0x4000ab81a8180594ull, 0x400030bab5b05045ull, 0x3000000b8aa85845ull,
    0x2000000000975879ull, 0x3000000375359039ull, 0x3000000751710870ull, 0x2000000000753351ull,
    0x300000021a759879ull, 0x400037503505921aull, 0x400025a758528208ull, 0x30000007533525a2ull,
    0x30000002b3987597ull, 0x4000b72029279759ull, 0x4000751871810b32ull, 0x300000051771b12bull,
    0x4000b3a31a758859ull, 0x50aba010b7905075ull, 0x507570805a30b0abull, 0x20000000005b75abull,
    0x100000000000056aull, 0x20000000006a5380ull, 0x20000000006a5109ull, 0x30000006a5891381ull,
    0x2000000000162561ull, 0x3000000803621561ull, 0x3000000620609569ull, 0x4000823625285895ull,
    0x200000000056ab32ull, 0x300000056a02b80bull, 0x30000006a5b32910ull, 0x4000b892b92916a5ull,
    0x3000000315356b36ull, 0x40006b51505b0b80ull, 0x40009505606306b3ull, 0x300000089bb96956ull,
    0x20000000008746a5ull, 0x3000000a56374034ull, 0x30000007486a5091ull, 0x400049737179156aull,
    0x3000000874156216ull, 0x4000743403625521ull, 0x4000620560509748ull, 0x5962695923497937ull,
    0x300000056a4872b3ull, 0x4000b720242746a5ull, 0x40006a5b32874910ull, 0x56a54b7b492b9129ull,
    0x40006b51535b3748ull, 0x5b404b7b016b5b15ull, 0x574836b630560950ull, 0x40009b7974b96956ull,
    0x2000000000a4694aull, 0x3000000380a946a4ull, 0x300000004606a10aull, 0x4000a16468618138ull,
    0x3000000462421941ull, 0x4000462942921803ull, 0x2000000000624420ull, 0x3000000624428238ull,
    0x300000032b46a94aull, 0x40006a4a94b82280ull, 0x4000a164606102b3ull, 0x51b8b12184a16146ull,
    0x400036b319639469ull, 0x514641916b0181b8ull, 0x30000004600636b3ull, 0x200000000086b846ull,
    0x3000000a98a876a7ull, 0x4000a76a907a0370ull, 0x40000818717a176aull, 0x300000037117a76aull,
    0x4000768981861621ull, 0x5937390976192962ull, 0x3000000206607087ull, 0x2000000000276237ull,
    0x400076898a86ab32ull, 0x57a9a76790b72702ull, 0x5b32a767a1871081ull, 0x400017616a71b12bull,
    0x563136b619768698ull, 0x200000000076b190ull, 0x400006b0b3607087ull, 0x10000000000006b7ull,
    0x1000000000000b67ull, 0x200000000067b803ull, 0x200000000067b910ull, 0x300000067b138918ull,
    0x20000000007b621aull, 0x30000007b6803a21ull, 0x30000007b69a2092ull, 0x400089a38a3a27b6ull,
    0x2000000000726327ull, 0x3000000026067807ull, 0x3000000910732672ull, 0x4000678891681261ull,
    0x300000073171a67aull, 0x4000801781a7167aull, 0x40007a69a0a70730ull, 0x30000009a88a7a67ull,
    0x200000000068b486ull, 0x3000000640603b63ull, 0x3000000109648b68ull, 0x400063b139369649ull,
    0x30000001a28b6486ull, 0x4000640b60b03a21ull, 0x40009a2920b648b4ull, 0x536463b34923a39aull,
    0x3000000264248328ull, 0x2000000000264240ull, 0x4000834642432091ull, 0x3000000642241491ull,
    0x40001a6648168318ull, 0x300000040660a01aull, 0x539a9303a6834364ull, 0x20000000004a649aull,
    0x2000000000b67594ull, 0x300000067b594380ull, 0x3000000b67045105ull, 0x400051345343867bull,
    0x3000000b6721a459ull, 0x4000594380a217b6ull, 0x4000204a24a45b67ull, 0x567b25a523453843ull,
    0x3000000945267327ull, 0x4000786260680459ull, 0x4000045051673263ull, 0x5851584812786826ull,
    0x400073167161a459ull, 0x5459078701671a61ull, 0x5a737a6a305a4a04ull, 0x4000a84a458a7a67ull,
    0x300000098b9b6596ull, 0x4000590650360b63ull, 0x4000b65510b508b0ull, 0x30000001355363b6ull,
    0x400065b8b9b59a21ull, 0x5a21965690b603b0ull, 0x552025a50865b58bull, 0x400035a3a25363b6ull,
    0x4000283265825985ull, 0x3000000260069659ull, 0x5826283865081851ull, 0x2000000000612651ull,
    0x5698965683a61631ull, 0x400006505960a01aull, 0x2000000000a65830ull, 0x100000000000065aull,
    0x2000000000b57a5bull, 0x300000003857ba5bull, 0x3000000091ba57b5ull, 0x40001381897ba57aull,
    0x300000015717b21bull, 0x4000b27571721380ull, 0x40007b2209729579ull, 0x5289823295b27257ull,
    0x3000000573532a52ull, 0x400052a578258028ull, 0x40002a37353a5109ull, 0x525752a278129289ull,
    0x2000000000573531ull, 0x3000000571170780ull, 0x3000000735539309ull, 0x2000000000795789ull,
    0x30000008ba8a5485ull, 0x400003bba50b5405ull, 0x400054aba8a48910ull, 0x541314943b54a4baull,
    0x40008548b2582152ull, 0x5b151b2b543b0b40ull, 0x558b8545b2950520ull, 0x20000000003b2549ull,
    0x4000483543253a52ull, 0x30000000244252a5ull, 0x5910854583a532a3ull, 0x40002492914252a5ull,
    0x3000000153358548ull, 0x2000000000501540ull, 0x4000530509358548ull, 0x1000000000000549ull,
    0x3000000ba9b947b4ull, 0x4000ba97b9794380ull, 0x4000b470414b1ba1ull, 0x54bab474a1843413ull,
    0x4000219b294b97b4ull, 0x53801b2b197b9479ull, 0x300000004224b47bull, 0x400042343824b47bull,
    0x4000947732972a92ull, 0x570207872a4797a9ull, 0x5a040a1a472a3a73ull, 0x20000000004782a1ull,
    0x3000000317714194ull, 0x4000178180714194ull, 0x2000000000347304ull, 0x1000000000000784ull,
    0x20000000008ba8a9ull, 0x3000000a9bb93903ull, 0x3000000ba88a0a10ull, 0x2000000000a3ba13ull,
    0x30000008b99b1b21ull, 0x40009b2921b93903ull, 0x2000000000b08b20ull, 0x1000000000000b23ull,
    0x300000098aa82832ull, 0x20000000002902a9ull, 0x40008a1810a82832ull, 0x10000000000002a1ull,
    0x2000000000819831ull, 0x1000000000000190ull, 0x1000000000000830ull, 0x0000000000000000ull,
};

// A cut edge joins corners of different sign (mc_tables.py:25-42 restated).
__device__ __forceinline__ unsigned mc_edge_mask(unsigned cube) {
  unsigned m = 0;
#pragma unroll
  for (int e = 0; e < 12; ++e)
    m |= (((cube >> kMcEdge[e][0]) ^ (cube >> kMcEdge[e][1])) & 1u) << e;
  return m;
}

// Neighbour index of an offset (dx, dy, dz) in {0,1}^3 (0 = the block itself),
// in meshing.py:38-47's order: +x, +y, +z, +xy, +xz, +yz, +xyz.
__device__ __forceinline__ int mc_nb_index(int dx, int dy, int dz) {
  const int code = dx | (dy << 1) | (dz << 2);
  // code: 1 x, 2 y, 4 z, 3 xy, 5 xz, 6 yz, 7 xyz  ->  1..7 as listed above
  constexpr int map[8] = {0, 1, 2, 4, 3, 5, 6, 7};
  return map[code];
}

// Hash tables of the other shards of a hash-sharded volume (device
// pointers valid here: the same device, or peers mapped over NVLink by
// CUDA IPC).  Marching cubes borrows the +x / +y / +z neighbours of a block
// (meshing.py:112-147); on a sharded volume a neighbour may live on another
// shard, so its corners are read from that shard's pool directly.
struct MeshPeer {
  const int* heads;
  const long long* keys;
  const int* next;
  const double* pool;
  long long buckets;
};
struct MeshPeers {
  MeshPeer p[kMaxShards];
  int count;  // shards (1: every neighbour is local)
  int self;
};

__device__ __forceinline__ int peer_find(const MeshPeer& P, long long key) {
  int n = __ldcg(&P.heads[block_hash_of_key(key, P.buckets)]);
  while (n >= 0) {
    if (__ldcg(&P.keys[n]) == key) return n;
    n = __ldcg(&P.next[n]);
  }
  return -1;
}

// The block itself and its seven +axis neighbours (block base pointers, null
// when absent), looked up once per CTA.
__device__ __forceinline__ void mc_neighbours(const Table& T, const MeshPeers& mp, long long key,
                                              int slot, const double** nb) {
  if (threadIdx.x < 8) {
    const double* ptr = T.pool + static_cast<size_t>(slot) * kBlockDoubles;
    if (threadIdx.x > 0) {
      constexpr int off[8][3] = {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1},
                                 {1, 1, 0}, {1, 0, 1}, {0, 1, 1}, {1, 1, 1}};
      long long bx, by, bz;
      unpack_key(key, bx, by, bz);
      bx += off[threadIdx.x][0];
      by += off[threadIdx.x][1];
      bz += off[threadIdx.x][2];
      const long long lim = kPackBias;  // packed coordinates must stay in 21 bits
      ptr = nullptr;
      if (bx < lim && by < lim && bz < lim) {
        const long long k = pack_key(bx, by, bz);
        const int o = mp.count > 1 ? key_owner(k, mp.count) : mp.self;
        if (o == mp.self) {
          const int s = chain_find(T, ld_acquire(&T.heads[block_hash_of_key(k, T.buckets)]), -1, k);
          if (s >= 0) ptr = T.pool + static_cast<size_t>(s) * kBlockDoubles;
        } else {
          const int s = peer_find(mp.p[o], k);
          if (s >= 0) ptr = mp.p[o].pool + static_cast<size_t>(s) * kBlockDoubles;
        }
      }
    }
    nb[threadIdx.x] = ptr;
  }
}

constexpr int kMcThreads = 128;  // four consecutive cells per thread
constexpr int kMcCells = kBlockVoxels / kMcThreads;
constexpr int kMcPad = 9;        // padded corner grid (meshing.py:112-146)
constexpr int kMcPadN = kMcPad * kMcPad * kMcPad;

// Padded position (x, y, z) in 0..8: owning block (neighbour index) and voxel.
__device__ __forceinline__ const double* mc_pad_source(const double* const* nb, int x, int y,
                                                       int z, int& voxel) {
  voxel = (x & 7) + 8 * (y & 7) + 64 * (z & 7);
  return nb[mc_nb_index(x >> 3, y >> 3, z >> 3)];
}

// Stage D and W of the 9x9x9 padded grid in shared memory (coalesced along
// x; an absent neighbour's corners read as W = 0, unobserved).
__device__ __forceinline__ void mc_stage(const double* const* nb, double* s_d, double* s_w) {
  for (int j = threadIdx.x; j < kMcPadN; j += blockDim.x) {
    int voxel;
    const double* blk =
        mc_pad_source(nb, j % kMcPad, (j / kMcPad) % kMcPad, j / (kMcPad * kMcPad), voxel);
    s_d[j] = blk ? blk[voxel] : 0.0;
    s_w[j] = blk ? blk[kBlockVoxels + voxel] : 0.0;
  }
}

__device__ __forceinline__ int mc_pad_index(int l, int corner) {
  const int x = (l & 7) + kMcCorner[corner][0], y = ((l >> 3) & 7) + kMcCorner[corner][1],
            z = (l >> 6) + kMcCorner[corner][2];
  return (z * kMcPad + y) * kMcPad + x;
}

// Case of cell l (meshing.py:157-164): 0 when not live.
__device__ __forceinline__ unsigned mc_case(const double* s_d, const double* s_w, int l,
                                            bool& live) {
  unsigned cube = 0;
  bool observed = true;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int j = mc_pad_index(l, i);
    observed = observed && s_w[j] > 0.0;
    cube |= (s_d[j] < 0.0 ? 1u : 0u) << i;
  }
  live = observed && mc_edge_mask(cube) != 0;
  return cube;
}

// Pass 1: vertices and triangles per block (sorted order).
__global__ void __launch_bounds__(kMcThreads, 8) k_mesh_count(Table T, MeshPeers mp,
                                                           const long long* keys,
                                                           const int* slots, long long n,
                                                           long long* nv, long long* nt) {
  __shared__ const double* nb[8];
  __shared__ double s_d[kMcPadN], s_w[kMcPadN];
  __shared__ int s_v[kMcThreads / 32], s_t[kMcThreads / 32];
  for (long long b = blockIdx.x; b < n; b += gridDim.x) {
    mc_neighbours(T, mp, keys[b], slots[b], nb);
    __syncthreads();
    mc_stage(nb, s_d, s_w);
    __syncthreads();
    int v = 0, t = 0;
#pragma unroll
    for (int q = 0; q < kMcCells; ++q) {
      bool live;
      const unsigned cube = mc_case(s_d, s_w, threadIdx.x * kMcCells + q, live);
      v += live ? __popc(mc_edge_mask(cube)) : 0;
      t += live ? static_cast<int>(kMcTriangles[cube] >> 60) : 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      v += __shfl_xor_sync(kFull, v, o);
      t += __shfl_xor_sync(kFull, t, o);
    }
    if ((threadIdx.x & 31) == 0) {
      s_v[threadIdx.x >> 5] = v;
      s_t[threadIdx.x >> 5] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      long long sv = 0, st = 0;
      for (int i = 0; i < kMcThreads / 32; ++i) {
        sv += s_v[i];
        st += s_t[i];
      }
      nv[b] = sv;
      nt[b] = st;
    }
    __syncthreads();
  }
}

// Pass 2: the block's vertices, colours and triangles at its offsets.  Each
// live cell lists its (cell, cut edge) and (cell, triangle) entries in shared
// memory at its prefix; the CTA then writes the block's contiguous output
// ranges one vertex / triangle per thread (coalesced stores).
__global__ void __launch_bounds__(kMcThreads, 6) k_mesh_emit(Table T, MeshPeers mp,
                                                          const long long* keys,
                                                          const int* slots, long long n,
                                                          const long long* v_off,
                                                          const long long* t_off, double vs,
                                                          double* verts, double* cols,
                                                          long long* tris) {
  __shared__ const double* nb[8];
  __shared__ double s_d[kMcPadN], s_w[kMcPadN];
  __shared__ unsigned short s_vlist[kBlockVoxels * 12];  // cell << 4 | edge
  __shared__ unsigned short s_tlist[kBlockVoxels * 5];   // cell << 3 | triangle
  __shared__ int s_vpre[kBlockVoxels];
  __shared__ unsigned char s_cube[kBlockVoxels];
  __shared__ int s_v[kMcThreads / 32], s_t[kMcThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (long long b = blockIdx.x; b < n; b += gridDim.x) {
    const long long key = keys[b];
    mc_neighbours(T, mp, key, slots[b], nb);
    __syncthreads();
    mc_stage(nb, s_d, s_w);
    __syncthreads();
    // this thread's cells l0 .. l0 + kMcCells - 1 (consecutive: l order)
    const int l0 = threadIdx.x * kMcCells;
    unsigned cubes[kMcCells];
    int nvc[kMcCells], ntc[kMcCells], sv = 0, st = 0;
#pragma unroll
    for (int q = 0; q < kMcCells; ++q) {
      bool live;
      cubes[q] = mc_case(s_d, s_w, l0 + q, live);
      nvc[q] = live ? __popc(mc_edge_mask(cubes[q])) : 0;
      ntc[q] = live ? static_cast<int>(kMcTriangles[cubes[q]] >> 60) : 0;
      sv += nvc[q];
      st += ntc[q];
    }
    // exclusive prefix over threads (warp scan + warp totals)
    int iv = sv, it = st;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(kFull, iv, o), c = __shfl_up_sync(kFull, it, o);
      if (lane >= o) {
        iv += a;
        it += c;
      }
    }
    if (lane == 31) {
      s_v[warp] = iv;
      s_t[warp] = it;
    }
    __syncthreads();
    int wv = 0, wt = 0, tv = 0, tt = 0;
    for (int i = 0; i < kMcThreads / 32; ++i) {
      if (i < warp) {
        wv += s_v[i];
        wt += s_t[i];
      }
      tv += s_v[i];
      tt += s_t[i];
    }
    int vpre = wv + iv - sv, tpre = wt + it - st;
#pragma unroll
    for (int q = 0; q < kMcCells; ++q) {
      const int l = l0 + q;
      s_vpre[l] = vpre;
      s_cube[l] = static_cast<unsigned char>(cubes[q]);
      if (nvc[q]) {
        const unsigned edges = mc_edge_mask(cubes[q]);
        int r = vpre;
        for (int e = 0; e < 12; ++e)
          if ((edges >> e) & 1u) s_vlist[r++] = static_cast<unsigned short>((l << 4) | e);
        for (int k = 0; k < ntc[q]; ++k)
          s_tlist[tpre + k] = static_cast<unsigned short>((l << 3) | k);
      }
      vpre += nvc[q];
      tpre += ntc[q];
    }
    __syncthreads();
    const long long vb = v_off[b], tb = t_off[b];
    long long bx, by, bz;
    unpack_key(key, bx, by, bz);
    for (int j = threadIdx.x; j < tv; j += kMcThreads) {
      const int cell = s_vlist[j] >> 4, e = s_vlist[j] & 15;
      const int a = kMcEdge[e][0], c = kMcEdge[e][1];
      const double da = s_d[mc_pad_index(cell, a)], db = s_d[mc_pad_index(cell, c)];
      const double den = da - db;
      const double t = den == 0.0 ? 0.5 : da / den;  // meshing.py:180-182
      const int x = cell & 7, y = (cell >> 3) & 7, z = cell >> 6;
      // corner v0 centre: (anchor + 0.5) * vs (meshing.py:190-192)
      const double base[3] = {(static_cast<double>(x + bx * kBlockSide) + 0.5) * vs,
                              (static_cast<double>(y + by * kBlockSide) + 0.5) * vs,
                              (static_cast<double>(z + bz * kBlockSide) + 0.5) * vs};
      int va, vc;  // both corners observed: their blocks exist
      const double* pa_blk =
          mc_pad_source(nb, x + kMcCorner[a][0], y + kMcCorner[a][1], z + kMcCorner[a][2], va);
      const double* pc_blk =
          mc_pad_source(nb, x + kMcCorner[c][0], y + kMcCorner[c][1], z + kMcCorner[c][2], vc);
      const long long vi = vb + j;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double pa = base[k] + (kMcCorner[a][k] ? vs : 0.0);
        const double pb = base[k] + (kMcCorner[c][k] ? vs : 0.0);
        verts[3 * vi + k] = pa + t * (pb - pa);
        const double ca = pa_blk[(2 + k) * kBlockVoxels + va];
        const double cb = pc_blk[(2 + k) * kBlockVoxels + vc];
        cols[3 * vi + k] = ca + t * (cb - ca);
      }
    }
    for (int j = threadIdx.x; j < tt; j += kMcThreads) {
      const int cell = s_tlist[j] >> 3, k = s_tlist[j] & 7;
      const unsigned cb = s_cube[cell];
      const unsigned em = mc_edge_mask(cb);
      const unsigned long long tl = kMcTriangles[cb];
      const long long v0 = vb + s_vpre[cell];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const int e = static_cast<int>((tl >> (4 * (3 * k + i))) & 0xf);
        tris[3 * (tb + j) + i] = v0 + __popc(em & ((1u << e) - 1u));
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// weld (meshing.py:248-276) on the device: key = rint(v / tol) per axis (numpy's
// round-half-even), rows sorted lexicographically by a stable LSD radix sort
// (z, then y, then x keys, carrying the vertex index, so equal keys keep index
// order and a segment's first entry is its lowest index -- np.unique's
// return_index), the first vertex of each segment kept, triangles remapped
// and collapsed ones dropped in order.

__global__ void k_weld_keys(const double* __restrict__ v, long long n, double tol,
                            long long* __restrict__ kx, long long* __restrict__ ky,
                            long long* __restrict__ kz, int* __restrict__ idx) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    kx[i] = __double2ll_rn(v[3 * i] / tol);
    ky[i] = __double2ll_rn(v[3 * i + 1] / tol);
    kz[i] = __double2ll_rn(v[3 * i + 2] / tol);
    idx[i] = static_cast<int>(i);
  }
}

__global__ void k_weld_gather(const long long* __restrict__ src, const int* __restrict__ perm,
                              long long n, long long* __restrict__ dst) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    dst[i] = src[perm[i]];
}

__global__ void k_weld_flags(const long long* __restrict__ kx, const long long* __restrict__ ky,
                             const long long* __restrict__ kz, const int* __restrict__ perm,
                             long long n, int* __restrict__ flag) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    int f = 1;
    if (i > 0) {
      const int a = perm[i], b = perm[i - 1];
      f = kx[a] != kx[b] || ky[a] != ky[b] || kz[a] != kz[b];
    }
    flag[i] = f;
  }
}

// seg = inclusive scan of flag (segment id + 1)
__global__ void k_weld_scatter(const int* __restrict__ perm, const int* __restrict__ flag,
                               const int* __restrict__ seg, long long n,
                               const double* __restrict__ v, const double* __restrict__ c,
                               double* __restrict__ vo, double* __restrict__ co,
                               int* __restrict__ inverse) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int src = perm[i], u = seg[i] - 1;
    inverse[src] = u;
    if (flag[i]) {
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        vo[3 * static_cast<long long>(u) + k] = v[3 * static_cast<long long>(src) + k];
        co[3 * static_cast<long long>(u) + k] = c[3 * static_cast<long long>(src) + k];
      }
    }
  }
}

__global__ void k_weld_tris(const long long* __restrict__ t, long long nt,
                            const int* __restrict__ inverse, long long* __restrict__ tr,
                            int* __restrict__ keep) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < nt;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long a = inverse[t[3 * i]], b = inverse[t[3 * i + 1]], c = inverse[t[3 * i + 2]];
    tr[3 * i] = a;
    tr[3 * i + 1] = b;
    tr[3 * i + 2] = c;
    keep[i] = a != b && b != c && a != c;
  }
}

// pos = inclusive scan of keep
__global__ void k_weld_compact(const long long* __restrict__ tr, const int* __restrict__ keep,
                               const int* __restrict__ pos, long long nt,
                               long long* __restrict__ out) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < nt;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    if (!keep[i]) continue;
    const long long o = pos[i] - 1;
#pragma unroll
    for (int k = 0; k < 3; ++k) out[3 * o + k] = tr[3 * i + k];
  }
}

// ---------------------------------------------------------------------------
// nn_min_d2 (the reference plugin's evaluation kernel, _kernels_cy.pyx:111-129):
// per query the minimum over all points of (dx*dx + dy*dy) + dz*dz, IEEE f64
// without contraction (the min itself is exact, so the point order is free).
// Points stream through shared memory in tiles; each thread owns two queries.

constexpr int kNnThreads = 256;
constexpr int kNnTile = 1024;  // points per shared-memory tile (24 KB)

__global__ void __launch_bounds__(kNnThreads) k_nn_min_d2(const double* __restrict__ q, long long n,
                                                          const double* __restrict__ pts,
                                                          long long m, double* __restrict__ out) {
  __shared__ double sp[3][kNnTile];
  const long long i0 = (static_cast<long long>(blockIdx.x) * kNnThreads + threadIdx.x) * 2;
  double qx[2], qy[2], qz[2], best[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const long long i = i0 + k < n ? i0 + k : 0;
    qx[k] = n ? q[3 * i] : 0.0;
    qy[k] = n ? q[3 * i + 1] : 0.0;
    qz[k] = n ? q[3 * i + 2] : 0.0;
    best[k] = CUDART_INF;
  }
  for (long long base = 0; base < m; base += kNnTile) {
    const int cnt = static_cast<int>(m - base < kNnTile ? m - base : kNnTile);
    __syncthreads();
    for (int j = threadIdx.x; j < 3 * cnt; j += kNnThreads) {
      const double v = pts[3 * base + j];
      sp[j % 3][j / 3] = v;
    }
    __syncthreads();
    for (int j = 0; j < cnt; ++j) {
      const double px = sp[0][j], py = sp[1][j], pz = sp[2][j];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const double dx = qx[k] - px, dy = qy[k] - py, dz = qz[k] - pz;
        double d2 = dx * dx + dy * dy;
        d2 = d2 + dz * dz;
        best[k] = d2 < best[k] ? d2 : best[k];
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 2; ++k)
    if (i0 + k < n) out[i0 + k] = best[k];
}

}  // namespace rf
