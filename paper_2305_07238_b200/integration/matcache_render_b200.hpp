// matcache_render_b200.hpp — extras of the B200 drop-in beyond the
// reference's tracer.hpp (which it implements; see matcache_render_b200.cpp).
#pragma once

#include "matcache/cache.hpp"

namespace matcache {

/// render(scene, config, &cache) keeps a device table standing in for
/// `cache` (seeded from it on every call, its inserts replayed back into it
/// after the call); this frees that device table. Optional: tables are
/// otherwise reused for the process's lifetime.
void b200_release_cache(const MaterialCache* cache);

}  // namespace matcache
