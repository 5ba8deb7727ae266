// Global GLL numbering without the 72M-key sort (host, native C++).
//
// The reference numbers nodes by sorting one NodeKey per local node
// (mesh.cpp:287-350): [0,vid] < [1,a,b,param] < [2,origin,xn,yn*(n+1)+s,t]
// < [3,e,node]. Because each key class sorts by entity first, the rank of a
// key has a closed form once the entities themselves are ranked:
//   vertex      -> rank of vid among referenced vertex ids
//   edge node   -> NVu + rankE(a,b)*(n-1) + (param-1)      (a<b, param from a)
//   face node   -> NVu + NEd*(n-1) + rankF(o,xn,yn)*(n-1)^2 + (s-1)*(n-1) + (t-1)
//   interior    -> NVu + NEd*(n-1) + NF*(n-1)^2 + e*(n-1)^3 + local interior rank
// where (o,xn,yn,s,t) is the canonical face frame of face_node_key
// (mesh.cpp:260-281): o = min corner id, xn = the smaller of o's two in-face
// neighbours. Only the entity lists are sorted (12 edges + 6 faces per
// element instead of (n+1)^3 48-byte keys), so this is O(NE log NE + N).
// Bit-exactness against the reference is checked in tests/test_host_setup.py
// (108 meshes, and cfg2 entry for entry in the slow test_numbering_bit_exact_cfg2).
//
// Also derived here: the Dirichlet mask (mesh.cpp:369-383) and the face slots
// of the extended (n+3)^3 subdomain numbering (sub_l2g, mesh.cpp:385-451).
#include <algorithm>
#include <numeric>
#include <thread>

#include "setup.hpp"
#include "setup_parallel.hpp"

namespace hxb {

int surface_slot_count(int np) { return np * np * np - (np - 2) * (np - 2) * (np - 2); }

// Rank of local node (i,j,k) among the element-surface nodes in ascending
// local-index order ((k*np+j)*np+i); -1 for element-interior nodes.
int surface_slot_of(int np, int i, int j, int k)
{
  const int n = np - 1;
  const int mid = 4 * np - 4;  // surface nodes per interior k-layer
  if (k == 0) return j * np + i;
  if (k == n) return np * np + (np - 2) * mid + j * np + i;
  const int base = np * np + (k - 1) * mid;
  if (j == 0) return base + i;
  if (j == n) return base + np + 2 * (np - 2) + i;
  if (i == 0) return base + np + 2 * (j - 1);
  if (i == n) return base + np + 2 * (j - 1) + 1;
  return -1;
}

namespace {

struct FaceKey {
  gid o, xn, yn;
  bool operator<(const FaceKey& b) const
  {
    if (o != b.o) return o < b.o;
    if (xn != b.xn) return xn < b.xn;
    return yn < b.yn;
  }
  bool operator==(const FaceKey& b) const { return o == b.o && xn == b.xn && yn == b.yn; }
};

// Face frame of element face (frozen axis a at side s): c[u][v] corner grid
// over axes a1=(a+1)%3 (u) and a2=(a+2)%3 (v), as in mesh.cpp:322-336.
struct FaceFrame {
  FaceKey key;
  int x0, y0, swap;
};

FaceFrame face_frame(const std::array<gid, 8>& conn, int a, int side)
{
  const int a1 = (a + 1) % 3, a2 = (a + 2) % 3;
  gid c[2][2];
  for (int u = 0; u < 2; ++u)
    for (int v = 0; v < 2; ++v) {
      int bits[3];
      bits[a] = side;
      bits[a1] = u;
      bits[a2] = v;
      c[u][v] = conn[hex_corner(bits[0], bits[1], bits[2])];
    }
  int x0 = 0, y0 = 0;
  for (int u = 0; u < 2; ++u)
    for (int v = 0; v < 2; ++v)
      if (c[u][v] < c[x0][y0]) {
        x0 = u;
        y0 = v;
      }
  const gid n0 = c[1 - x0][y0];  // xn when swap = 0
  const gid n1 = c[x0][1 - y0];  // xn when swap = 1
  FaceFrame f;
  f.x0 = x0;
  f.y0 = y0;
  f.swap = n0 < n1 ? 0 : 1;
  f.key = {c[x0][y0], f.swap ? n1 : n0, f.swap ? n0 : n1};
  return f;
}

inline std::uint64_t edge_key(gid a, gid b)
{
  const gid lo = std::min(a, b), hi = std::max(a, b);
  return (static_cast<std::uint64_t>(static_cast<std::uint32_t>(lo)) << 32) | static_cast<std::uint32_t>(hi);
}

// Edge list of the reference cube: interior axis a, the other two bits (u,v).
struct EdgeDef {
  int a, lo_corner, hi_corner;
};
std::array<EdgeDef, 12> make_edges()
{
  std::array<EdgeDef, 12> t{};
  int q = 0;
  for (int a = 0; a < 3; ++a)
    for (int v = 0; v < 2; ++v)
      for (int u = 0; u < 2; ++u) {
        int lo[3], hi[3];
        lo[a] = 0;
        hi[a] = 1;
        lo[(a + 1) % 3] = hi[(a + 1) % 3] = u;
        lo[(a + 2) % 3] = hi[(a + 2) % 3] = v;
        t[q++] = {a, hex_corner(lo[0], lo[1], lo[2]), hex_corner(hi[0], hi[1], hi[2])};
      }
  return t;
}
const std::array<EdgeDef, 12> kEdges = make_edges();

// Which of kEdges an edge node belongs to: interior axis a, fixed bits of the other two axes.
inline int edge_index(int a, int bit_a1, int bit_a2)
{
  // make_edges enumerates (a, v over a2, u over a1)
  return a * 4 + bit_a2 * 2 + bit_a1;
}

}  // namespace

Numbering build_numbering(const HexMesh& mesh, int order)
{
  const int n = order, np = n + 1;
  const gid ne = mesh.num_elements(), nv = mesh.num_vertices();
  Numbering num;
  num.order = n;

  // (0) referenced vertices in id order
  std::vector<std::uint8_t> used(nv, 0);
  for (const auto& el : mesh.elements)
    for (gid v : el) {
      if (v < 0 || v >= nv) throw HxbError(2, "element references vertex id out of range");
      used[v] = 1;
    }
  num.vertex_rank.assign(nv, -1);
  gid nvu = 0;
  for (gid v = 0; v < nv; ++v)
    if (used[v]) num.vertex_rank[v] = nvu++;
  num.num_vertex_nodes = nvu;

  // (1) unique edges ordered by (min id, max id)
  setup_phase("numbering: edges");
  std::vector<std::uint64_t> edges(static_cast<std::size_t>(ne) * 12);
  parallel_for(ne, [&](gid b, gid en) {
    for (gid e = b; e < en; ++e)
      for (int q = 0; q < 12; ++q)
        edges[static_cast<std::size_t>(e) * 12 + q] =
            edge_key(mesh.elements[e][kEdges[q].lo_corner], mesh.elements[e][kEdges[q].hi_corner]);
  });
  std::vector<std::uint64_t> uedges = edges;
  parallel_sort(uedges, std::less<std::uint64_t>());
  uedges.erase(std::unique(uedges.begin(), uedges.end()), uedges.end());
  num.num_edges = static_cast<gid>(uedges.size());
  std::vector<gid> erank(edges.size());
  parallel_for(ne, [&](gid b, gid en) {
    for (std::size_t i = static_cast<std::size_t>(b) * 12; i < static_cast<std::size_t>(en) * 12; ++i)
      erank[i] = static_cast<gid>(std::lower_bound(uedges.begin(), uedges.end(), edges[i]) - uedges.begin());
  });
  edges.clear();
  edges.shrink_to_fit();

  // (2) unique faces ordered by canonical frame (origin, xn, yn)
  setup_phase("numbering: faces");
  std::vector<FaceFrame> frames(static_cast<std::size_t>(ne) * 6);
  parallel_for(ne, [&](gid b, gid en) {
    for (gid e = b; e < en; ++e)
      for (int f = 0; f < 6; ++f) frames[static_cast<std::size_t>(e) * 6 + f] = face_frame(mesh.elements[e], f / 2, f % 2);
  });
  std::vector<std::pair<FaceKey, std::int64_t>> fk(frames.size());
  for (std::size_t i = 0; i < frames.size(); ++i) fk[i] = {frames[i].key, static_cast<std::int64_t>(i)};
  parallel_sort(fk, [](const std::pair<FaceKey, std::int64_t>& x, const std::pair<FaceKey, std::int64_t>& y) {
    if (x.first == y.first) return x.second < y.second;
    return x.first < y.first;
  });
  std::vector<gid> frank(frames.size());
  num.face_nbr_elem.assign(frames.size(), -1);
  num.face_nbr_face.assign(frames.size(), -1);
  gid nf = 0;
  for (std::size_t i = 0; i < fk.size();) {
    std::size_t j = i;
    while (j < fk.size() && fk[j].first == fk[i].first) ++j;
    if (j - i > 2) throw HxbError(2, "non-conforming mesh: face shared by more than two elements");
    for (std::size_t q = i; q < j; ++q) frank[fk[q].second] = nf;
    if (j - i == 2) {
      const auto a = fk[i].second, b = fk[i + 1].second;
      num.face_nbr_elem[a] = static_cast<gid>(b / 6);
      num.face_nbr_face[a] = static_cast<std::int8_t>(b % 6);
      num.face_nbr_elem[b] = static_cast<gid>(a / 6);
      num.face_nbr_face[b] = static_cast<std::int8_t>(a % 6);
    }
    ++nf;
    i = j;
  }
  num.num_faces = nf;
  fk.clear();
  fk.shrink_to_fit();

  const std::int64_t nm1 = n - 1;
  const std::int64_t surf_total = nvu + static_cast<std::int64_t>(num.num_edges) * nm1 +
                                  static_cast<std::int64_t>(nf) * nm1 * nm1;
  const std::int64_t total = surf_total + static_cast<std::int64_t>(ne) * nm1 * nm1 * nm1;
  if (total > 0x7fffffffLL) throw HxbError(1, "mesh too large for int32 global ids");
  num.num_surface_global = static_cast<gid>(surf_total);
  num.num_global = static_cast<gid>(total);

  // (3) per-element surface slots
  setup_phase("numbering: surface ids");
  const int nsurf = surface_slot_count(np);
  num.l2g_surf.assign(static_cast<std::size_t>(ne) * nsurf, -1);
  parallel_for(ne, [&](gid b, gid en) {
    for (gid e = b; e < en; ++e) {
      const auto& conn = mesh.elements[e];
      gid* out = num.l2g_surf.data() + static_cast<std::size_t>(e) * nsurf;
      for (int k = 0; k < np; ++k)
        for (int j = 0; j < np; ++j)
          for (int i = 0; i < np; ++i) {
            const int s = surface_slot_of(np, i, j, k);
            if (s < 0) continue;
            const int idx[3] = {i, j, k};
            const int pos[3] = {i == 0 ? 0 : (i == n ? 2 : 1), j == 0 ? 0 : (j == n ? 2 : 1),
                                k == 0 ? 0 : (k == n ? 2 : 1)};
            const int nint = (pos[0] == 1) + (pos[1] == 1) + (pos[2] == 1);
            gid g;
            if (nint == 0) {
              g = num.vertex_rank[conn[hex_corner(i / n, j / n, k / n)]];
            } else if (nint == 1) {
              const int a = pos[0] == 1 ? 0 : (pos[1] == 1 ? 1 : 2);
              const int a1 = (a + 1) % 3, a2 = (a + 2) % 3;
              const int q = edge_index(a, idx[a1] / n, idx[a2] / n);
              gid va = conn[kEdges[q].lo_corner], vb = conn[kEdges[q].hi_corner];
              int param = idx[a];
              if (va > vb) param = n - param;
              g = static_cast<gid>(nvu + static_cast<std::int64_t>(erank[static_cast<std::size_t>(e) * 12 + q]) * nm1 +
                                   (param - 1));
            } else {
              const int a = pos[0] != 1 ? 0 : (pos[1] != 1 ? 1 : 2);
              const int a1 = (a + 1) % 3, a2 = (a + 2) % 3;
              const int f = 2 * a + idx[a] / n;
              const FaceFrame& fr = frames[static_cast<std::size_t>(e) * 6 + f];
              const int p = idx[a1], qq0 = idx[a2];
              const int pp = fr.x0 ? n - p : p;
              const int qq = fr.y0 ? n - qq0 : qq0;
              const int ss = fr.swap ? qq : pp;
              const int tt = fr.swap ? pp : qq;
              g = static_cast<gid>(nvu + static_cast<std::int64_t>(num.num_edges) * nm1 +
                                   static_cast<std::int64_t>(frank[static_cast<std::size_t>(e) * 6 + f]) * nm1 * nm1 +
                                   (ss - 1) * nm1 + (tt - 1));
            }
            out[s] = g;
          }
    }
  });

  // (4) Dirichlet mask from tagged faces (mesh.cpp:369-383)
  setup_phase("numbering: dirichlet mask");
  num.dirichlet_mask.assign(num.num_global, 0);
  for (const auto& bf : mesh.boundary_faces) {
    if (bf.tag != 0) continue;
    if (bf.element < 0 || bf.element >= ne || bf.face < 0 || bf.face > 5)
      throw HxbError(1, "boundary face out of range");
    const int a = bf.face / 2, s = bf.face % 2;
    for (int v = 0; v < np; ++v)
      for (int u = 0; u < np; ++u) {
        int ijk[3];
        ijk[a] = s ? n : 0;
        ijk[(a + 1) % 3] = u;
        ijk[(a + 2) % 3] = v;
        const int sl = surface_slot_of(np, ijk[0], ijk[1], ijk[2]);
        num.dirichlet_mask[num.l2g_surf[static_cast<std::size_t>(bf.element) * nsurf + sl]] = 1;
      }
  }

  // (5) sub_l2g face slots (mesh.cpp:419-450): neighbour's first interior layer
  setup_phase("numbering: sub_face");
  // The shared face's canonical frame (step 2) is the same in both elements,
  // so a face node's coordinates in the neighbour follow from the two frames:
  // e's (u, v) -> canonical (ss, tt) -> the neighbour's (u2, v2), then one
  // layer inward. Each mapped face node is checked against the neighbour's
  // copy of it (same global id).
  const std::size_t fs = static_cast<std::size_t>(np) * np;
  num.sub_face.assign(static_cast<std::size_t>(ne) * 6 * fs, -1);
  parallel_for(ne, [&](gid b, gid en) {
    auto node_gid = [&](gid el, const int (&ijk)[3]) -> gid {
      const int sl = surface_slot_of(np, ijk[0], ijk[1], ijk[2]);
      if (sl >= 0) return num.l2g_surf[static_cast<std::size_t>(el) * nsurf + sl];
      return static_cast<gid>(num.num_surface_global + static_cast<std::int64_t>(el) * nm1 * nm1 * nm1 +
                              ((ijk[2] - 1) * nm1 + (ijk[1] - 1)) * nm1 + (ijk[0] - 1));
    };
    for (gid e = b; e < en; ++e) {
      for (int f = 0; f < 6; ++f) {
        const gid e2 = num.face_nbr_elem[static_cast<std::size_t>(e) * 6 + f];
        if (e2 < 0) continue;
        const int f2 = num.face_nbr_face[static_cast<std::size_t>(e) * 6 + f];
        const FaceFrame& fr = frames[static_cast<std::size_t>(e) * 6 + f];
        const FaceFrame& fr2 = frames[static_cast<std::size_t>(e2) * 6 + f2];
        const int a = f / 2, s = f % 2, a2 = f2 / 2, s2 = f2 % 2;
        gid* out = num.sub_face.data() + (static_cast<std::size_t>(e) * 6 + f) * fs;
        for (int v = 0; v < np; ++v)
          for (int u = 0; u < np; ++u) {
            const int pp = fr.x0 ? n - u : u, qq = fr.y0 ? n - v : v;
            const int ss = fr.swap ? qq : pp, tt = fr.swap ? pp : qq;
            const int pp2 = fr2.swap ? tt : ss, qq2 = fr2.swap ? ss : tt;
            const int u2 = fr2.x0 ? n - pp2 : pp2, v2 = fr2.y0 ? n - qq2 : qq2;
            int ijk[3], ijk2[3];
            ijk[a] = s ? n : 0;
            ijk[(a + 1) % 3] = u;
            ijk[(a + 2) % 3] = v;
            ijk2[a2] = s2 ? n : 0;
            ijk2[(a2 + 1) % 3] = u2;
            ijk2[(a2 + 2) % 3] = v2;
            if (node_gid(e, ijk) != node_gid(e2, ijk2))
              throw HxbError(2, "global node has no copy in expected neighbor element");
            ijk2[a2] += s2 ? -1 : 1;
            out[v * np + u] = node_gid(e2, ijk2);
          }
      }
    }
  });
  return num;
}

void element_l2g(const Numbering& num, int ne_total, gid e, gid* out)
{
  (void)ne_total;
  const int n = num.order, np = n + 1;
  const int nsurf = surface_slot_count(np);
  const gid* surf = num.l2g_surf.data() + static_cast<std::size_t>(e) * nsurf;
  const std::int64_t nm1 = n - 1;
  const std::int64_t ibase = num.num_surface_global + static_cast<std::int64_t>(e) * nm1 * nm1 * nm1;
  int l = 0;
  for (int k = 0; k < np; ++k)
    for (int j = 0; j < np; ++j)
      for (int i = 0; i < np; ++i, ++l) {
        const int s = surface_slot_of(np, i, j, k);
        out[l] = s >= 0 ? surf[s]
                        : static_cast<gid>(ibase + ((k - 1) * nm1 + (j - 1)) * nm1 + (i - 1));
      }
}

}  // namespace hxb
