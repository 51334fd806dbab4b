// Writes a test pattern through include/fgs_io.hpp's write_image (PNG and PPM) and a PLY round
// trip through save_ply / load_ply; tests/test_image_io.py decodes and checks the files.
#include <cstdio>
#include <cstdlib>
#include <string>

#include "../../include/fgs_io.hpp"

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  const std::string dir = argv[1];
  fgs::Image img;
  img.width = 300;   // > 65535 bytes of scanlines: several stored deflate blocks
  img.height = 97;
  img.pixels.resize(static_cast<size_t>(img.width) * img.height * 3);
  for (size_t i = 0; i < img.pixels.size(); ++i) img.pixels[i] = static_cast<float>((i % 517) / 512.0 - 0.004);
  // 0.5 * 255 = 127.5 exactly: rounds to the even 128; out-of-range and NaN values clamp
  img.pixels[0] = 0.5f;
  img.pixels[1] = -3.0f;
  img.pixels[2] = 7.0f;
  img.pixels[3] = std::nanf("");
  fgs::io::write_image(img, dir + "/pattern.png");
  fgs::io::write_image(img, dir + "/pattern.ppm");
  FILE* f = std::fopen((dir + "/pattern.f32").c_str(), "wb");
  std::fwrite(img.pixels.data(), 4, img.pixels.size(), f);
  std::fclose(f);
  try {
    fgs::io::write_image(img, dir + "/pattern.bmp");
    return 3;
  } catch (const std::runtime_error& e) {
    std::printf("%s\n", e.what());
  }
  return 0;
}
