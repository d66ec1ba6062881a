// Driver for tests/test_obj_io.py: parses an OBJ file with a material table
// through include/roomray_b200_io.hpp and writes the result (or the error)
// as raw arrays / a status file.
//   obj_parity <obj> <materials.json> <out_dir>
#include <fstream>
#include <iostream>
#include <string>
#include <vector>

#include "roomray_b200_io.hpp"

namespace rb = roomray_b200;

template <typename T>
static void write_all(const std::string& path, const std::vector<T>& v) {
  std::ofstream f(path, std::ios::binary);
  f.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(T)));
}

int main(int argc, char** argv) {
  if (argc != 4) return 2;
  const std::string out = argv[3];
  std::ofstream status(out + "/status.txt");
  try {
    const auto table = rb::load_material_table(argv[2]);
    rb::LoadReport rep;
    const rb::TriangleMesh mesh = rb::load_obj(argv[1], table, &rep);
    std::vector<double> v, a;
    std::vector<int32_t> f;
    for (const auto& p : mesh.vertices) v.insert(v.end(), {p.x, p.y, p.z});
    for (const auto& t : mesh.faces) f.insert(f.end(), {t.a, t.b, t.c, t.material_id});
    for (const auto& m : mesh.materials) a.insert(a.end(), m.absorption.begin(), m.absorption.end());
    write_all(out + "/vertices.f64", v);
    write_all(out + "/faces.i32", f);
    write_all(out + "/alpha.f64", a);
    status << "ok " << rep.degenerate_skipped << " " << rep.vertex_count << " " << rep.face_count << "\n";
  } catch (const rb::ObjParseError& e) {
    status << "parse " << e.line() << "\n" << e.what() << "\n";
  } catch (const rb::UnresolvedMaterialError& e) {
    status << "material 0\n" << e.what() << "\n";
  } catch (const std::exception& e) {
    status << "other 0\n" << e.what() << "\n";
  }
  return 0;
}
