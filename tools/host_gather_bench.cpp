// host_gather_bench.cpp -- characterise the GPU box's host side for the
// host-slab path (rocp_stream_consume_range_host): memory bandwidth, random
// 8-byte load throughput (4 KB vs transparent huge pages) and fibre-gather
// strategies on the configs[1] window shape (1000 x 1000 x 25 slabs, S = 600).
// Build: g++ -O3 -march=native -pthread tools/host_gather_bench.cpp -o tools/host_gather_bench
#include <sys/mman.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static double* alloc(size_t n, bool huge) {
    const size_t H = size_t(2) << 20;
    size_t len = (n * 8 + H - 1) / H * H;
    void* p = mmap(nullptr, len + H, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    uintptr_t a = (uintptr_t(p) + H - 1) & ~(uintptr_t(H) - 1);
    madvise((void*)a, len, huge ? MADV_HUGEPAGE : MADV_NOHUGEPAGE);
    return (double*)a;
}

template <class F>
static void par(int nt, F f) {
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t) th.emplace_back(f, t, nt);
    for (auto& x : th) x.join();
}

int main(int argc, char** argv) {
    const int64_t I1 = 1000, I2 = 1000, B = 25, S = 600;
    const int nbat = argc > 1 ? atoi(argv[1]) : 36;
    const int64_t slice = I1 * I2, slab = slice * B, total = slab * nbat;
    const int hw = int(std::thread::hardware_concurrency());
    printf("hw threads %d, window %.2f GB\n", hw, total * 8e-9);
    for (int huge = 0; huge < 2; ++huge) {
        double* x = alloc(size_t(total), huge);
        double t0 = now();
        par(hw, [&](int t, int nt) {
            for (int64_t k = int64_t(t) * total / nt; k < int64_t(t + 1) * total / nt; ++k) x[k] = double(k & 1023);
        });
        double t1 = now();
        FILE* f = fopen("/proc/meminfo", "r");
        char line[256];
        long anon_huge = 0;
        while (f && fgets(line, sizeof line, f))
            if (!strncmp(line, "AnonHugePages:", 14)) anon_huge = atol(line + 14);
        if (f) fclose(f);
        printf("[huge=%d] first-touch fill %.1f GB/s, AnonHugePages %ld MB\n", huge, total * 8e-9 / (t1 - t0),
               anon_huge / 1024);
        // streaming read bandwidth
        for (int nt : {1, 8, hw}) {
            std::atomic<double> sink{0};
            t0 = now();
            par(nt, [&](int t, int n) {
                double s = 0;
                for (int64_t k = int64_t(t) * total / n; k < int64_t(t + 1) * total / n; k += 8) s += x[k];
                sink = sink + s;
            });
            t1 = now();
            printf("  read bw %2d thr: %.1f GB/s\n", nt, total * 8e-9 / (t1 - t0));
        }
        // per-batch sample bases (mode-2 fibres: i1 + t*slice, stride I1)
        std::mt19937_64 g(7);
        std::vector<int64_t> base2(size_t(nbat * S)), baset(size_t(nbat * S));
        for (int b = 0; b < nbat; ++b)
            for (int64_t c = 0; c < S; ++c) {
                base2[size_t(b * S + c)] = int64_t(b) * slab + int64_t(g() % I1) + int64_t(g() % B) * slice;
                baset[size_t(b * S + c)] = int64_t(b) * slab + int64_t(g() % I1) + int64_t(g() % I2) * I1;
            }
        std::vector<double> out(size_t(nbat * S * I2));
        const int64_t acc = int64_t(nbat) * S * (I2 + B);
        auto report = [&](const char* name, int nt, double dt) {
            printf("  %-34s %2d thr: %7.2f ms  %6.0f M acc/s\n", name, nt, dt * 1e3, acc / dt * 1e-6);
        };
        for (int nt : {8, hw, 2 * hw}) {
            for (int D : {0, 8, 32}) {
                t0 = now();
                par(nt, [&](int t, int n) {
                    for (int64_t k = t; k < int64_t(nbat) * S; k += n) {
                        const double* s2 = x + base2[size_t(k)];
                        double* o = out.data() + k * I2;
                        for (int64_t i = 0; i < I2; ++i) {
                            if (D) __builtin_prefetch(s2 + (i + D) * I1, 0, 0);
                            o[i] = s2[i * I1];
                        }
                        const double* st = x + baset[size_t(k)];
                        double acc2 = 0;
                        for (int64_t i = 0; i < B; ++i) acc2 += st[i * slice];
                        o[0] += acc2 * 0;
                    }
                });
                t1 = now();
                char nm[64];
                snprintf(nm, sizeof nm, "per-fibre prefetch D=%d", D);
                report(nm, nt, t1 - t0);
            }
            for (int C : {16, 64}) {
                t0 = now();
                par(nt, [&](int t, int n) {
                    std::vector<int64_t> ord(size_t(S));
                    for (int64_t k0 = int64_t(t) * C; k0 < int64_t(nbat) * S; k0 += int64_t(n) * C) {
                        const int64_t k1 = std::min<int64_t>(int64_t(nbat) * S, k0 + C);
                        for (int64_t i = 0; i < I2; ++i)
                            for (int64_t k = k0; k < k1; ++k) out[size_t(k * I2 + i)] = x[base2[size_t(k)] + i * I1];
                        for (int64_t k = k0; k < k1; ++k) {
                            double a2 = 0;
                            for (int64_t i = 0; i < B; ++i) a2 += x[baset[size_t(k)] + i * slice];
                            out[size_t(k * I2)] += a2 * 0;
                        }
                    }
                });
                t1 = now();
                char nm[64];
                snprintf(nm, sizeof nm, "row-interleaved C=%d", C);
                report(nm, nt, t1 - t0);
            }
        }
        // real host-slab gather: 3 stages per batch (temporal stride slice, mode 1 contiguous,
        // mode 2 stride I1), row-tiled destination xs_offset(i, c) = ((i>>5)*S + c)*32 + (i&31),
        // 6-batch sub-windows, tasks of F fibres claimed from an atomic counter.
        if (huge) {
            const int64_t per_b = (B + 31) / 32 * 32 * S + I1 * S + I2 * S;
            double* hx = alloc(size_t(per_b * nbat), true);
            std::memset(hx, 0, size_t(per_b * nbat) * 8);
            std::vector<int64_t> base1(size_t(nbat * S));
            for (int b = 0; b < nbat; ++b)
                for (int64_t c = 0; c < S; ++c)
                    base1[size_t(b * S + c)] = int64_t(b) * slab + int64_t(g() % I2) * I1 + int64_t(g() % B) * slice;
            auto xs = [&](int64_t i, int64_t c) { return ((i >> 5) * S + c) * 32 + (i & 31); };
            for (int variant = 0; variant < 4; ++variant)
                for (int F : {4, 16, 64}) {
                    const int nt = hw;
                    t0 = now();
                    for (int b0 = 0; b0 < nbat; b0 += 6) {
                        const int b1 = std::min(nbat, b0 + 6);
                        struct T {
                            int b, st;
                            int64_t c0, c1;
                        };
                        std::vector<T> tasks;
                        for (int pass = 0; pass < 2; ++pass)
                            for (int b = b0; b < b1; ++b)
                                for (int st = 0; st < 3; ++st) {
                                    if ((st == 1) != (pass == 1)) continue;
                                    for (int64_t c0 = 0; c0 < S; c0 += F) tasks.push_back(T{b, st, c0, std::min(S, c0 + F)});
                                }
                        std::atomic<size_t> next{0};
                        par(nt, [&](int, int) {
                            double tmp[1024];
                            for (size_t k = next++; k < tasks.size(); k = next++) {
                                const T& tk = tasks[size_t(k)];
                                const int64_t I = tk.st == 0 ? B : tk.st == 1 ? I1 : I2;
                                const int64_t ms = tk.st == 0 ? slice : tk.st == 1 ? 1 : I1;
                                const int64_t* bs = tk.st == 0 ? baset.data() : tk.st == 1 ? base1.data() : base2.data();
                                const int64_t so = tk.st == 0 ? 0 : tk.st == 1 ? (B + 31) / 32 * 32 * S : (B + 31) / 32 * 32 * S + I1 * S;
                                double* dst = hx + int64_t(tk.b) * per_b + so;
                                for (int64_t c = tk.c0; c < tk.c1; ++c) {
                                    const double* f = x + bs[size_t(tk.b * S + c)];
                                    if (ms == 1) {
                                        for (int64_t i0 = 0; i0 < I; i0 += 32)
                                            std::memcpy(dst + xs(i0, c), f + i0, size_t(std::min<int64_t>(32, I - i0)) * 8);
                                    } else if (variant == 0) {
                                        for (int64_t i0 = 0; i0 < I; i0 += 32) {
                                            double* o = dst + xs(i0, c);
                                            const int64_t n = std::min<int64_t>(32, I - i0);
                                            const double* fi = f + i0 * ms;
                                            for (int64_t i = 0; i < n; ++i) o[i] = fi[i * ms];
                                        }
                                    } else if (variant == 1) {
                                        for (int64_t i = 0; i < I; ++i) tmp[i] = f[i * ms];
                                        for (int64_t i0 = 0; i0 < I; i0 += 32)
                                            std::memcpy(dst + xs(i0, c), tmp + i0, size_t(std::min<int64_t>(32, I - i0)) * 8);
                                    } else if (variant == 2) {
#pragma GCC novector
                                        for (int64_t i = 0; i < I; ++i) tmp[i] = f[i * ms];
                                        for (int64_t i0 = 0; i0 < I; i0 += 32)
                                            std::memcpy(dst + xs(i0, c), tmp + i0, size_t(std::min<int64_t>(32, I - i0)) * 8);
                                    } else {
                                        // 4 fibres interleaved
                                        for (int64_t i = 0; i < I; ++i) dst[xs(i, c)] = f[i * ms];
                                    }
                                }
                            }
                        });
                    }
                    t1 = now();
                    printf("  real gather variant %d F=%2d %2d thr: %7.2f ms\n", variant, F, nt, (t1 - t0) * 1e3);
                }
            munmap(hx, 0);
        }
        munmap(x, (size_t(total) * 8 + (size_t(2) << 20) - 1) / (size_t(2) << 20) * (size_t(2) << 20));
    }
    return 0;
}
