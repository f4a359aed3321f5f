// adapter_demo.cpp — the INTEGRATION.md caller, compiled as C++17 against include/isocull_b200.hpp
// (+ the C ABI it wraps) and linked with libisocull_b200.so.  Test program of
// tests/test_cpp_adapter.py:
//   adapter_demo cpu  : host-only surface (errors, config validation, camera, IoU, composite)
//   adapter_demo gpu  : one PIFu frame (16 -> 64, 64x64 render) + a config-0 extraction, printed
//                       as one JSON line for the test to compare with the Python face
#include <cstdio>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "isocull_b200.hpp"

namespace ib = isocull_b200;

static int cpu_mode() {
    int fails = 0;
    auto expect = [&](bool ok, const char* what) {
        if (!ok) {
            std::fprintf(stderr, "FAIL: %s\n", what);
            ++fails;
        }
    };
    // validate_config messages and exception types follow localize.hpp:47-55
    ib::AlgoConfig bad;
    bad.coarsest_cells = 1;
    try {
        ib::validate_config(bad);
        expect(false, "coarsest 1 accepted");
    } catch (const std::invalid_argument& e) {
        expect(std::string(e.what()) == "config: coarsest cells must be >= 2", "message");
    }
    // CameraSpec::from_angles(90, 0): view z = -world x (render.hpp:36-45)
    ib::CameraSpec cam = ib::CameraSpec::from_angles(90, 0);
    ib::Vec3 v = cam.world_to_view({1, 0, 0});
    expect(std::abs(v.z + 1.0) < 1e-12 && std::abs(v.x) < 1e-12, "yaw 90 maps +x to -z");
    ib::Vec3 w = cam.view_to_world(v);
    expect(std::abs(w.x - 1.0) < 1e-12, "view_to_world inverts world_to_view");
    // compare_iou on host arrays, both-empty rule (localize.hpp:377-387)
    std::vector<std::uint8_t> a{1, 1, 0, 0}, b{1, 0, 1, 0}, z(4, 0);
    expect(std::abs(ib::compare_iou(a, b) - 1.0 / 3.0) < 1e-15, "iou");
    expect(ib::compare_iou(z, z) == 1.0, "iou of two empty volumes");
    try {
        ib::compare_iou(a, std::vector<std::uint8_t>(3));
        expect(false, "iou size mismatch accepted");
    } catch (const std::invalid_argument&) {
    }
    // composite (render.hpp:284-291), C++ and C ABI forms agree
    ib::RenderedImage img;
    img.width = 2;
    img.height = 1;
    img.rgb = {{1, 0, 0}, {0, 1, 0}};
    img.mask = {1, 0};
    std::vector<ib::Vec3> back{{0, 0, 1}, {0, 0, 1}};
    std::vector<ib::Vec3> out = ib::composite(img, back);
    expect(out[0].x == 1 && out[1].z == 1, "composite");
    float rgb[6] = {1, 0, 0, 0, 1, 0}, bd[6] = {0, 0, 1, 0, 0, 1}, o[6];
    std::uint8_t m[2] = {1, 0};
    ib::check(icg_composite(rgb, m, 2, bd, 2, o));
    expect(o[0] == 1 && o[5] == 1, "icg_composite");
    expect(icg_composite(rgb, m, 2, bd, 3, o) == ICG_EINVAL, "icg_composite mismatch");
    // no device on a CPU host: the library reports it, it never fakes a device
    int n = -1;
    ib::check(icg_device_count(&n));
    if (n == 0) {
        try {
            ib::Context ctx(0);
            expect(false, "context without a device");
        } catch (const std::runtime_error&) {
        }
    }
    std::printf("{\"mode\": \"cpu\", \"fails\": %d, \"devices\": %d}\n", fails, n);
    return fails ? 1 : 0;
}

static int gpu_mode() {
    // seeded inputs: capsules(42), feature map(1000) 256x32x32, weights(7, 8)
    std::vector<icg_primitive> caps(15);
    ib::check(icg_gen_capsules(42, 15, caps.data()));
    const int C = 256, H = 32, W = 32;
    std::vector<float> fmap((size_t)C * H * W);
    ib::check(icg_gen_normals(1000, fmap.size(), fmap.data()));
    ib::Context ctx(0);
    for (int which = 0; which < 2; ++which) {
        std::int32_t outs[5], ins[5], skip;
        std::size_t nw, nb;
        ib::check(icg_mlp_shape(which, outs, ins, &skip, &nw, &nb));
        std::vector<float> wf(nw), bf(nb);
        ib::check(icg_gen_mlp(which == 0 ? 7 : 8, which, wf.data(), bf.data()));
        std::vector<std::vector<float>> ws, bs;
        std::size_t wo = 0, bo = 0;
        for (int l = 0; l < 5; ++l) {
            ws.emplace_back(wf.begin() + wo, wf.begin() + wo + (size_t)outs[l] * ins[l]);
            bs.emplace_back(bf.begin() + bo, bf.begin() + bo + outs[l]);
            wo += (size_t)outs[l] * ins[l];
            bo += outs[l];
        }
        ctx.set_mlp(which, ws, bs);
    }
    ib::Field field = ib::Field::pifu(fmap.data(), C, H, W, caps);
    ib::AlgoConfig cfg;
    cfg.coarsest_cells = 16;
    cfg.target_level = 2;
    auto fr = ib::frame(ctx, field, cfg, ib::CameraSpec::from_angles(90, 0), 64, 64);
    const ib::ExtractionResult& r = fr.first;
    const ib::RenderedImage& im = fr.second;
    double vsum = 0.0, rgbsum = 0.0;
    for (float x : r.grid.values) vsum += x;
    for (const ib::Vec3& c : im.rgb) rgbsum += c.x + c.y + c.z;
    int covered = 0;
    for (auto mk : im.mask) covered += mk;
    // config-0 analytic field through extract / extract_brute_force / compare_iou / acceleration_factor
    ib::Field an = ib::Field::analytic(caps, 0.02);
    ib::AlgoConfig c0;
    c0.coarsest_cells = 8;
    c0.target_level = 3;
    ib::ExtractionResult p = ib::extract_progressive(ctx, an, c0);
    ib::ExtractionResult bt = ib::extract_brute_force(ctx, an, c0);
    const double iou = ib::compare_iou(p.binarized, bt.binarized);
    // the reference renderer (view-aligned, render.hpp:244-280) on the analytic field with a
    // constant texture, and the Fig. 4 octree baseline through the same extract()
    icg_texture_rule tex{};
    tex.kind = ICG_TEXTURE_CONSTANT;
    tex.color[0] = 0.25, tex.color[1] = 0.5, tex.color[2] = 0.75;
    ib::Field tan = ib::Field::analytic(caps, 0.02, tex);
    ib::RenderedImage rv = ib::render_view(ctx, tan, ib::CameraSpec::from_angles(30, 20), c0);
    int rv_cov = 0;
    for (auto mk : rv.mask) rv_cov += mk;
    ib::AlgoConfig oc = c0;
    oc.variant = ib::Variant::octree_threshold;
    oc.threshold = 0.12;
    ib::ExtractionResult ot = ib::extract(ctx, an, oc);
    ib::TriangleMesh mesh = ib::marching_cubes(ctx, p.grid);
    // invalid config -> std::invalid_argument from the library itself
    bool threw = false;
    try {
        ib::AlgoConfig big = c0;
        big.target_level = 8;
        icg_algo_config cc = big.to_c();
        icg_extraction e{};
        ib::check(icg_extract(ctx.get(), an.get(), &cc, &e));
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    std::printf("{\"mode\": \"gpu\", \"evals\": [%llu, %llu, %llu], \"total\": %llu, \"value_sum\": %.17g, "
                "\"covered\": %d, \"rgb_sum\": %.17g, \"c0_evals\": [%llu, %llu, %llu, %llu], \"iou\": %.17g, "
                "\"accel\": %.17g, \"invalid_threw\": %s, \"rv_covered\": %d, \"rv_calls\": %llu, "
                "\"octree_evals\": %llu, \"mesh_vertices\": %zu, \"mesh_triangles\": %zu}\n",
                (unsigned long long)r.evals_per_level[0], (unsigned long long)r.evals_per_level[1],
                (unsigned long long)r.evals_per_level[2], (unsigned long long)r.total_evals, vsum, covered, rgbsum,
                (unsigned long long)p.evals_per_level[0], (unsigned long long)p.evals_per_level[1],
                (unsigned long long)p.evals_per_level[2], (unsigned long long)p.evals_per_level[3], iou,
                ib::acceleration_factor(p, bt), threw ? "true" : "false", rv_cov,
                (unsigned long long)rv.oracle_calls, (unsigned long long)ot.total_evals, mesh.vertices.size(),
                mesh.triangles.size());
    return 0;
}

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "cpu";
    try {
        return mode == "gpu" ? gpu_mode() : cpu_mode();
    } catch (const std::exception& e) {
        std::fprintf(stderr, "exception: %s\n", e.what());
        return 3;
    }
}
