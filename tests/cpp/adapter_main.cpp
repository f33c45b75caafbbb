// Test driver of the C++ adapter (include/dabd_gpu.hpp): a host program written
// in the reference's vocabulary (sim.hpp / scene.hpp) stepping the B200 path.
//
//   adapter_main scene NAME                 print the built body table (no GPU):
//                                           n, then per body q0[6] and mass as %a
//   adapter_main io DIR                     snapshot / metrics round trip (no GPU)
//   adapter_main reference NAME FRAMES DIR  run_reference -> DIR/frame_%04d.bin
//   adapter_main distributed NAME FRAMES WORKERS DIR
//                                           run_distributed -> snapshots + metrics.csv
// Prints one JSON line of totals for the stepping modes.
#include <cstdio>
#include <cstdlib>
#include <string>

#include "dabd_gpu.hpp"

using namespace dabd::gpu;

static int cmd_scene(const std::string& name) {
    const SceneData sd = make_scenario(name);
    Scene sc(sd);
    std::printf("%d\n", sc.size());
    for (int b = 0; b < sc.size(); ++b) {
        for (double v : sc.initial_configs()[b]) std::printf("%a ", v);
        std::printf("%a\n", sc.mass()[b]);
    }
    return 0;
}

static int cmd_io(const std::string& dir) {
    std::filesystem::create_directories(dir);
    const std::vector<bool> is_static{true, false, false};
    Configs q{{0, 0, 1, 0, 0, 1}, {0.1, 0.2, 1, 1e-3, -1e-3, 1}, {-1.5, 2.25, 0.5, 0, 0, 2}};
    Configs qd{{0, 0, 0, 0, 0, 0}, {1, 2, 3, 4, 5, 6}, {-1, -2, -3, -4, -5, -6}};
    write_snapshot(frame_path(dir, 0), 0, is_static, q, qd);
    q[1][0] = 0.3;
    write_snapshot(frame_path(dir, 1), 1, is_static, q, qd);
    const Snapshot s = read_snapshot(frame_path(dir, 1));
    if (s.frame != 1 || s.ids.size() != 2 || s.ids[0] != 1 || s.q[0][0] != 0.3 || s.q_dot[1][5] != -6)
        return 2;
    Configs init{{7, 7, 1, 0, 0, 1}, {0, 0, 1, 0, 0, 1}, {0, 0, 1, 0, 0, 1}};
    const Trajectory t = load_trajectory(dir, init);
    if (t.q.size() != 2 || t.q[0][0][0] != 7 || t.q[1][1][0] != 0.3 || t.q_dot[1][2][0] != -1) return 3;
    if (std::abs(mse_to_reference(is_static, t.q[1], t.q[0]) - 0.04 / 12.0) > 1e-15) return 4;
    MetricsRow r;
    r.frame = 0;
    r.k = 2;
    r.r_inf = 1.5e-7;
    r.commit_row = true;
    r.dq_inf = {1e-6, 2e-6};
    r.newton_iters = {3, 4};
    write_metrics_csv(dir + "/metrics.csv", {r}, 2);
    std::printf("io ok\n");
    return 0;
}

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: adapter_main scene|io|reference|distributed ...\n");
        return 1;
    }
    const std::string mode = argv[1];
    try {
        if (mode == "scene") return cmd_scene(argv[2]);
        if (mode == "io") return cmd_io(argv[2]);
        if (mode == "reference" && argc == 5) {
            SceneData sd = make_scenario(argv[2]);
            sd.frames = std::atoi(argv[3]);
            const Trajectory t = run_reference(sd, argv[4]);
            std::printf("{\"mode\": \"reference\", \"frames\": %zu}\n", t.q.size());
            return 0;
        }
        if (mode == "distributed" && argc == 6) {
            SceneData sd = make_scenario(argv[2]);
            sd.frames = std::atoi(argv[3]);
            RunOptions opt;
            opt.workers = std::atoi(argv[4]);
            opt.out_dir = argv[5];
            opt.audit = true;
            const RunResult r = run_distributed(sd, opt);
            long admm = 0;
            for (const FrameStats& f : r.frames) admm += f.admm_iterations;
            std::printf("{\"mode\": \"distributed\", \"frames\": %zu, \"admm_iterations\": %ld, "
                        "\"metrics_rows\": %zu, \"intersection_violations\": %d}\n",
                        r.trajectory.q.size(), admm, r.metrics.size(), r.intersection_violations);
            return 0;
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 5;
    }
    std::fprintf(stderr, "bad arguments\n");
    return 1;
}
