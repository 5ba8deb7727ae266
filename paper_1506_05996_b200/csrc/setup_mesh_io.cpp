// Mesh file formats on either side of the solve, host C++.
//
//   read_msh / write_msh        Gmsh MSH 2.2 ASCII subset      mesh_io.cpp:49-145
//   read_native / write_native  "HXSM0001" compact binary      mesh_io.cpp:147-218
//   read_mesh_file / write_...  dispatch on ".msh"             mesh_io.cpp:220-232
//
// Behaviour follows the reference readers: sparse Gmsh node ids, foreign
// element types skipped, boundary quads matched to hexahedron faces through
// their sorted corner ids (physical tag 2 = Neumann, anything else Dirichlet),
// every element's Jacobian checked at the 27 reference points on the way in
// (check_jacobians, geometry.cpp:153-161). The parser is a single pass over
// the file image with from_chars (correctly rounded, like the reference's
// stream extraction) so meshes with millions of hexes load in seconds, and
// the binary reader checks the file length before allocating.
#include <algorithm>
#include <array>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <string>
#include <system_error>
#include <unordered_map>

#include "setup.hpp"

namespace hxb {

namespace {

constexpr int kEio = 6;  // HXB_EIO
constexpr char kMagic[8] = {'H', 'X', 'S', 'M', '0', '0', '0', '1'};

[[noreturn]] void io_error(const std::string& msg) { throw HxbError(kEio, msg); }

std::string slurp(const std::string& path)
{
  std::ifstream in(path, std::ios::binary);
  if (!in) io_error("cannot open mesh file " + path);
  in.seekg(0, std::ios::end);
  const std::streamoff n = in.tellg();
  in.seekg(0, std::ios::beg);
  std::string s(static_cast<std::size_t>(n < 0 ? 0 : n), '\0');
  in.read(s.data(), static_cast<std::streamsize>(s.size()));
  return s;
}

// Line cursor over the file image; tokens split on blanks/tabs/CR.
struct Lines {
  const char* p;
  const char* end;
  bool next(const char*& b, const char*& e)
  {
    if (p >= end) return false;
    b = p;
    const void* nl = std::memchr(p, '\n', static_cast<std::size_t>(end - p));
    e = nl ? static_cast<const char*>(nl) : end;
    p = nl ? e + 1 : end;
    return true;
  }
};

struct Tok {
  const char* p;
  const char* end;
  const std::string* path;
  void skip()
  {
    while (p < end && (*p == ' ' || *p == '\t' || *p == '\r')) ++p;
  }
  template <class T>
  T get()
  {
    skip();
    T v{};
    const auto r = std::from_chars(p, end, v);
    if (r.ec != std::errc()) io_error("malformed line in mesh file " + *path);
    p = r.ptr;
    return v;
  }
};

bool starts_with(const char* b, const char* e, const char* key)
{
  const std::size_t n = std::strlen(key);
  return static_cast<std::size_t>(e - b) >= n && std::memcmp(b, key, n) == 0;
}

using Quad = std::array<gid, 4>;

Quad sorted_quad(Quad q)
{
  std::sort(q.begin(), q.end());
  return q;
}

struct QuadHash {
  std::size_t operator()(const Quad& q) const
  {
    std::size_t h = 1469598103934665603ull;
    for (gid v : q) h = (h ^ static_cast<std::uint32_t>(v)) * 1099511628211ull;
    return h;
  }
};

// attach_boundary_quads (mesh_io.cpp:28-45): a face key maps to the LAST
// (element, face) that produced it, as the reference's map assignment does.
void attach_boundary_quads(HexMesh& mesh, const std::vector<std::pair<Quad, int>>& quads)
{
  if (quads.empty()) return;
  std::unordered_map<Quad, std::pair<gid, int>, QuadHash> face_of;
  face_of.reserve(6 * static_cast<std::size_t>(mesh.num_elements()));
  for (gid e = 0; e < mesh.num_elements(); ++e)
    for (int f = 0; f < 6; ++f) {
      Quad key{};
      for (int c = 0; c < 4; ++c) key[c] = mesh.elements[e][face_corners(f)[c]];
      face_of[sorted_quad(key)] = {e, f};
    }
  for (const auto& [verts, tag] : quads) {
    const auto it = face_of.find(sorted_quad(verts));
    if (it == face_of.end()) io_error("boundary quad does not match any hexahedron face");
    mesh.boundary_faces.push_back(
        {it->second.first, it->second.second, static_cast<std::uint8_t>(tag == 2 ? 1 : 0)});
  }
}

}  // namespace

HexMesh read_msh(const std::string& path)
{
  const std::string text = slurp(path);
  Lines lines{text.data(), text.data() + text.size()};
  HexMesh mesh;
  std::vector<std::pair<Quad, int>> quads;
  std::unordered_map<long long, gid> node_id;  // gmsh ids may be sparse
  const char *b, *e;
  auto need_line = [&] {
    if (!lines.next(b, e)) io_error("truncated mesh file " + path);
  };
  while (lines.next(b, e)) {
    if (starts_with(b, e, "$MeshFormat")) {
      need_line();
      Tok t{b, e, &path};
      double version = 0;
      t.skip();
      std::from_chars(t.p, t.end, version);
      if (version < 2.0 || version >= 3.0) io_error("unsupported MSH version in " + path);
      need_line();  // $EndMeshFormat
    } else if (starts_with(b, e, "$Nodes")) {
      need_line();
      const auto count = Tok{b, e, &path}.get<unsigned long long>();
      mesh.vertices.reserve(count);
      node_id.reserve(count);
      for (unsigned long long i = 0; i < count; ++i) {
        need_line();
        Tok t{b, e, &path};
        const long long id = t.get<long long>();
        const double x = t.get<double>(), y = t.get<double>(), z = t.get<double>();
        node_id[id] = mesh.num_vertices();
        mesh.vertices.push_back({x, y, z});
      }
      need_line();  // $EndNodes
    } else if (starts_with(b, e, "$Elements")) {
      need_line();
      const auto count = Tok{b, e, &path}.get<unsigned long long>();
      auto vertex = [&](long long nid) {
        const auto it = node_id.find(nid);
        if (it == node_id.end()) io_error("element references unknown node " + std::to_string(nid) + " in " + path);
        return it->second;
      };
      for (unsigned long long i = 0; i < count; ++i) {
        need_line();
        Tok t{b, e, &path};
        (void)t.get<long long>();
        const int type = t.get<int>(), ntags = t.get<int>();
        int physical = 0;
        for (int q = 0; q < ntags; ++q) {
          const int tag = t.get<int>();
          if (q == 0) physical = tag;
        }
        if (type == 5) {
          std::array<gid, 8> conn{};
          for (auto& v : conn) v = vertex(t.get<long long>());
          mesh.elements.push_back(conn);
        } else if (type == 3) {
          Quad verts{};
          for (auto& v : verts) v = vertex(t.get<long long>());
          quads.push_back({verts, physical});
        }  // other element types (points, lines) are skipped
      }
      need_line();  // $EndElements
    }
  }
  if (mesh.elements.empty()) io_error("no hexahedra found in " + path);
  attach_boundary_quads(mesh, quads);
  check_jacobians(mesh);
  return mesh;
}

void write_msh(const HexMesh& mesh, const std::string& path)
{
  std::FILE* f = std::fopen(path.c_str(), "w");
  if (!f) io_error("cannot write mesh file " + path);
  std::fprintf(f, "$MeshFormat\n2.2 0 8\n$EndMeshFormat\n$Nodes\n%zu\n", mesh.vertices.size());
  for (std::size_t v = 0; v < mesh.vertices.size(); ++v)
    std::fprintf(f, "%zu %.17g %.17g %.17g\n", v + 1, mesh.vertices[v][0], mesh.vertices[v][1], mesh.vertices[v][2]);
  std::fprintf(f, "$EndNodes\n$Elements\n%zu\n", mesh.elements.size() + mesh.boundary_faces.size());
  std::size_t id = 1;
  for (const auto& bf : mesh.boundary_faces) {  // tagged quads first, then the hexes (mesh_io.cpp:131-140)
    const int tag = bf.tag == 1 ? 2 : 1;
    std::fprintf(f, "%zu 3 2 %d %d", id++, tag, tag);
    for (int c : face_corners(bf.face)) std::fprintf(f, " %d", mesh.elements[bf.element][c] + 1);
    std::fputc('\n', f);
  }
  for (const auto& conn : mesh.elements) {
    std::fprintf(f, "%zu 5 2 0 0", id++);
    for (gid v : conn) std::fprintf(f, " %d", v + 1);
    std::fputc('\n', f);
  }
  std::fprintf(f, "$EndElements\n");
  if (std::fclose(f) != 0) io_error("cannot write mesh file " + path);
}

void write_native(const HexMesh& mesh, const std::string& path)
{
  const std::uint64_t nv = mesh.vertices.size(), ne = mesh.elements.size(), nb = mesh.boundary_faces.size();
  std::string img(8 + 24 + 24 * nv + 32 * ne + 12 * nb, '\0');
  char* p = img.data();
  auto put = [&](const void* src, std::size_t n) {
    std::memcpy(p, src, n);
    p += n;
  };
  put(kMagic, 8);
  const std::uint64_t counts[3] = {nv, ne, nb};
  put(counts, sizeof(counts));
  for (const auto& v : mesh.vertices) put(v.data(), 24);
  for (const auto& conn : mesh.elements) {
    std::uint32_t c[8];
    for (int i = 0; i < 8; ++i) c[i] = static_cast<std::uint32_t>(conn[i]);
    put(c, sizeof(c));
  }
  for (const auto& bf : mesh.boundary_faces) {
    const std::uint32_t rec[3] = {static_cast<std::uint32_t>(bf.element), static_cast<std::uint32_t>(bf.face),
                                  static_cast<std::uint32_t>(bf.tag)};
    put(rec, sizeof(rec));
  }
  std::ofstream out(path, std::ios::binary);
  if (!out) io_error("cannot write mesh file " + path);
  out.write(img.data(), static_cast<std::streamsize>(img.size()));
  if (!out) io_error("cannot write mesh file " + path);
}

HexMesh read_native(const std::string& path)
{
  const std::string img = slurp(path);
  if (img.size() < 8 || std::memcmp(img.data(), kMagic, 8) != 0) io_error(path + " is not a hexsem native mesh");
  if (img.size() < 32) io_error("truncated mesh file " + path);
  std::uint64_t counts[3];
  std::memcpy(counts, img.data() + 8, sizeof(counts));
  // length check before any allocation (a corrupt header cannot trigger a huge resize)
  const std::uint64_t limit = 1ull << 31;
  if (counts[0] >= limit || counts[1] >= limit || counts[2] >= limit ||
      img.size() < 32 + 24 * counts[0] + 32 * counts[1] + 12 * counts[2])
    io_error("truncated mesh file " + path);
  const char* p = img.data() + 32;
  HexMesh mesh;
  mesh.vertices.resize(counts[0]);
  for (auto& v : mesh.vertices) {
    std::memcpy(v.data(), p, 24);
    p += 24;
  }
  mesh.elements.resize(counts[1]);
  for (auto& conn : mesh.elements) {
    std::uint32_t c[8];
    std::memcpy(c, p, sizeof(c));
    p += sizeof(c);
    for (int i = 0; i < 8; ++i) {
      if (c[i] >= counts[0]) io_error("element references unknown vertex in " + path);
      conn[i] = static_cast<gid>(c[i]);
    }
  }
  mesh.boundary_faces.resize(counts[2]);
  for (auto& bf : mesh.boundary_faces) {
    std::uint32_t rec[3];
    std::memcpy(rec, p, sizeof(rec));
    p += sizeof(rec);
    if (rec[0] >= counts[1] || rec[1] > 5 || rec[2] > 1) io_error("boundary face record out of range in " + path);
    bf = {static_cast<gid>(rec[0]), static_cast<int>(rec[1]), static_cast<std::uint8_t>(rec[2])};
  }
  check_jacobians(mesh);
  return mesh;
}

namespace {
bool is_msh(const std::string& path) { return path.size() > 4 && path.compare(path.size() - 4, 4, ".msh") == 0; }
}  // namespace

HexMesh read_mesh_file(const std::string& path) { return is_msh(path) ? read_msh(path) : read_native(path); }

void write_mesh_file(const HexMesh& mesh, const std::string& path)
{
  if (is_msh(path))
    write_msh(mesh, path);
  else
    write_native(mesh, path);
}

}  // namespace hxb
