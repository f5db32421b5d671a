// Host-side (CPU) steps of the path that are sequential by definition, in
// C++ so they do not run at Python speed.  No device code.
//
// ft_wind_triangles: the consistent winding of the dual triangles
// (reference dual.py:284-313): from every not yet visited triangle in index
// order, a depth-first walk (explicit LIFO stack) over shared edges -- the
// triangle's edges in order (0-1, 1-2, 2-0), the triangles sharing an edge
// in ascending index -- flips each newly reached triangle that runs along
// the shared edge in the same direction as the one it was reached from.
// The visiting order is the reference's, so the result is identical also
// for a non-orientable configuration.

#include <algorithm>
#include <cstdint>
#include <utility>
#include <vector>

#include "fieldtess_cuda.h"

extern "C" int ft_wind_triangles(int64_t m, int32_t* tris) {
    if (m < 0 || (m > 0 && !tris)) return FT_ERR_ARG;
    if (m == 0) return FT_OK;
    int64_t base = 0;
    for (int64_t i = 0; i < 3 * m; ++i) base = std::max<int64_t>(base, tris[i]);
    base += 1;
    // undirected edge keys in (triangle, side) order, stably sorted: the
    // triangles of an edge come out in ascending index
    std::vector<std::pair<int64_t, int64_t>> ek((size_t)(3 * m));
    for (int64_t i = 0; i < m; ++i)
        for (int s = 0; s < 3; ++s) {
            const int64_t u = tris[3 * i + s], v = tris[3 * i + (s + 1) % 3];
            ek[(size_t)(3 * i + s)] = {std::min(u, v) * base + std::max(u, v), i};
        }
    std::stable_sort(ek.begin(), ek.end(),
                     [](const std::pair<int64_t, int64_t>& a, const std::pair<int64_t, int64_t>& b) {
                         return a.first < b.first;
                     });
    std::vector<char> seen((size_t)m, 0);
    std::vector<int64_t> stack;
    for (int64_t root = 0; root < m; ++root) {
        if (seen[(size_t)root]) continue;
        seen[(size_t)root] = 1;
        stack.push_back(root);
        while (!stack.empty()) {
            const int64_t cur = stack.back();
            stack.pop_back();
            const int32_t x[3] = {tris[3 * cur], tris[3 * cur + 1], tris[3 * cur + 2]};
            for (int s = 0; s < 3; ++s) {
                const int64_t u = x[s], v = x[(s + 1) % 3];
                const int64_t key = std::min(u, v) * base + std::max(u, v);
                auto lo = std::lower_bound(ek.begin(), ek.end(), std::make_pair(key, (int64_t)-1));
                for (auto it = lo; it != ek.end() && it->first == key; ++it) {
                    const int64_t other = it->second;
                    if (other == cur || seen[(size_t)other]) continue;
                    int32_t* y = tris + 3 * other;
                    if ((y[0] == u && y[1] == v) || (y[1] == u && y[2] == v) || (y[2] == u && y[0] == v))
                        std::swap(y[1], y[2]);          // (y0, y1, y2) -> (y0, y2, y1)
                    seen[(size_t)other] = 1;
                    stack.push_back(other);
                }
            }
        }
    }
    return FT_OK;
}
