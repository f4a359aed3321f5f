// io_host.cu — stream I/O of the C ABI: the reference's output writers (image.hpp:18-48,
// grid.hpp:199-222), byte-identical, for host buffers of the library's fp32 outputs.  Plain host
// C++ (no device work); errors map like the reference (invalid_argument -> ICG_EINVAL, I/O
// failure -> ICG_ERUNTIME).
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "icg_internal.h"

using namespace icg;

namespace {
int io_fail(const std::string& m, int code) {
    set_error(m);
    return code;
}
struct File {
    FILE* f;
    explicit File(const char* path, const char* mode) : f(std::fopen(path, mode)) {}
    ~File() {
        if (f) std::fclose(f);
    }
};
}  // namespace

extern "C" {

// write_ppm (image.hpp:18-33): P6, byte = lround(255 * clamp(v, 0, 1)) of each channel (as double)
int icg_write_ppm(const char* path, int width, int height, const float* rgb) {
    if (!path || width < 0 || height < 0 || (!rgb && width * height)) return io_fail("write_ppm: bad arguments", ICG_EINVAL);
    File out(path, "wb");
    if (!out.f) return io_fail(std::string("write_ppm: cannot open ") + path, ICG_ERUNTIME);
    std::fprintf(out.f, "P6\n%d %d\n255\n", width, height);
    const size_t n = (size_t)width * height * 3;
    std::vector<unsigned char> bytes(n);
    for (size_t i = 0; i < n; ++i) {
        const double v = rgb[i];
        const double c = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
        bytes[i] = (unsigned char)std::lround(255.0 * c);
    }
    if (std::fwrite(bytes.data(), 1, n, out.f) != n) return io_fail(std::string("write_ppm: write failed for ") + path, ICG_ERUNTIME);
    return ICG_OK;
}

// write_float_map (image.hpp:37-48): int32 width, height, then float32 values
int icg_write_float_map(const char* path, int width, int height, const float* values) {
    if (!path || width < 0 || height < 0 || (!values && width * height))
        return io_fail("write_float_map: bad arguments", ICG_EINVAL);
    File out(path, "wb");
    if (!out.f) return io_fail(std::string("write_float_map: cannot open ") + path, ICG_ERUNTIME);
    const int32_t hdr[2] = {width, height};
    const size_t n = (size_t)width * height;
    if (std::fwrite(hdr, 4, 2, out.f) != 2 || std::fwrite(values, 4, n, out.f) != n)
        return io_fail(std::string("write_float_map: write failed for ") + path, ICG_ERUNTIME);
    return ICG_OK;
}

// export_obj (mesh.hpp:159-172)
int icg_write_obj(const char* path, const double* v, uint64_t nv, const int32_t* t, uint64_t nt) {
    if (!path || (nv && !v) || (nt && !t)) return io_fail("export_obj: bad arguments", ICG_EINVAL);
    File out(path, "w");
    if (!out.f) return io_fail(std::string("export_obj: cannot open ") + path, ICG_ERUNTIME);
    std::fprintf(out.f, "# isocull mesh: %llu vertices, %llu triangles\n", (unsigned long long)nv, (unsigned long long)nt);
    for (uint64_t i = 0; i < nv; ++i) std::fprintf(out.f, "v %.9f %.9f %.9f\n", v[3 * i], v[3 * i + 1], v[3 * i + 2]);
    for (uint64_t i = 0; i < nt; ++i) std::fprintf(out.f, "f %d %d %d\n", t[3 * i] + 1, t[3 * i + 1] + 1, t[3 * i + 2] + 1);
    if (std::ferror(out.f)) return io_fail(std::string("export_obj: write failed for ") + path, ICG_ERUNTIME);
    return ICG_OK;
}

// dump_grid (grid.hpp:199-209): int32 level, int32 R, then (R+1)^3 float32 values x-fastest
int icg_dump_grid(const char* path, int level, int cells, const float* values) {
    if (!path || cells < 0 || !values) return io_fail("dump_grid: bad arguments", ICG_EINVAL);
    File out(path, "wb");
    if (!out.f) return io_fail(std::string("dump_grid: cannot open ") + path, ICG_ERUNTIME);
    const int32_t hdr[2] = {level, cells};
    const size_t n = ((size_t)cells + 1) * ((size_t)cells + 1) * ((size_t)cells + 1);
    if (std::fwrite(hdr, 4, 2, out.f) != 2 || std::fwrite(values, 4, n, out.f) != n)
        return io_fail(std::string("dump_grid: write failed for ") + path, ICG_ERUNTIME);
    return ICG_OK;
}

// load_grid_dump (grid.hpp:211-222): header always; values when `values` is non-null and holds
// `capacity` floats ((R+1)^3 needed, else ICG_ECAPACITY)
int icg_load_grid_dump(const char* path, int* level, int* cells, float* values, size_t capacity) {
    if (!path || !level || !cells) return io_fail("load_grid_dump: bad arguments", ICG_EINVAL);
    File in(path, "rb");
    if (!in.f) return io_fail(std::string("load_grid_dump: cannot open ") + path, ICG_ERUNTIME);
    int32_t hdr[2];
    if (std::fread(hdr, 4, 2, in.f) != 2) return io_fail(std::string("load_grid_dump: short header in ") + path, ICG_ERUNTIME);
    *level = hdr[0];
    *cells = hdr[1];
    if (!values) return ICG_OK;
    const size_t n = ((size_t)hdr[1] + 1) * ((size_t)hdr[1] + 1) * ((size_t)hdr[1] + 1);
    if (capacity < n) return io_fail("load_grid_dump: capacity too small", ICG_ECAPACITY);
    if (std::fread(values, 4, n, in.f) != n) return io_fail(std::string("load_grid_dump: short data in ") + path, ICG_ERUNTIME);
    return ICG_OK;
}

}  // extern "C"
